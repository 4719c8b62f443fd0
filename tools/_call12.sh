python -m pytest -q -m gpu tests/test_gpu_loopback.py -x -k "nradial4" 2>&1 | tail -5 > gpurun_out/gpu12.log
timeout 900 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_run.py > gpurun_out/memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck.log
