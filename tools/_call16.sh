for be in 2 3 4; do python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu --bin-every $be > gpurun_out/b16_be$be.json 2>&1; done
for mu in 2 8; do python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu --bin-every 3 --bin-mu $mu > gpurun_out/b16_be3_mu$mu.json 2>&1; done
