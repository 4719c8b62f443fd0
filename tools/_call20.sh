python -m pytest -q -m gpu tests/test_gpu_edge.py -k "push_computed or bin_keys" tests/test_gpu_parity.py 2>&1 | tail -3 > gpurun_out/gpu20.log
for v in "3 1" "3.5 1" "4 1" "3 0.5" "4 0.5"; do set -- $v; GTCP_RHO_CUT=$1 GTCP_DRIFT_CELLS=$2 python tools/prof_step.py --size A --steps 6 --warmup 3 --tag "rho$1_drift$2" >> gpurun_out/cut20.log 2>&1; done
