python -m pytest -q -m gpu tests/test_gpu_parity.py -k "push or step" 2>&1 | tail -2 > gpurun_out/gpu15.log
python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/b15_base.json 2>&1
python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --bin-every 1 > gpurun_out/b15_bin1.json 2>&1
python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --bin-every 3 > gpurun_out/b15_bin3.json 2>&1
