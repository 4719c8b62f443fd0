GTCP_PROFILE_BIN=1 python tools/prof_step.py --size A --steps 6 --warmup 3 > gpurun_out/bin18.log 2>&1
