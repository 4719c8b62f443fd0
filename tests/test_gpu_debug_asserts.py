"""Device-side bounds checks (compute-sanitizer is closed on this pool): the
library built with -DGTCP_DEBUG turns every DCHECK (shared-memory window
offsets of the deposit, global grid node indices, tile ranges) into a device
assert; a few full steps at T (2 and 8 planes) and at the class-A grid run
under it in a subprocess and must finish cleanly."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("args", [["T", "2", "12000"], ["T", "8", "40000"], ["A", "64", "1000000"]])
def test_steps_under_device_asserts(args):
    sys.path.insert(0, ROOT)
    from paper_1510_05546_b200 import _build
    lib = _build.build(debug=True)
    env = dict(os.environ, GTCP_LIB_PATH=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "debug_step.py")] + args, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "3 steps ok" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])
