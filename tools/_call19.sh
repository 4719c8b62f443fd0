for d in 1 1.5 2 3; do GTCP_DRIFT_CELLS=$d python tools/prof_step.py --size A --steps 6 --warmup 3 --tag drift$d >> gpurun_out/drift19.log 2>&1; done
