python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_grid_scale.py -x 2>&1 | tail -5 > gpurun_out/gpu4.log
python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/b4.json 2>&1
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_deposit_tiled -s 2 -c 1 -o gpurun_out/dep_r02b python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu4.log 2>&1
