python -m pytest -q -m gpu tests/test_gpu_edge.py -k "update_binning" 2>&1 | tail -5 > gpurun_out/gpu13.log
python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --charge-mode 2 > gpurun_out/b13_points.json 2>&1
python -m pytest -q -m gpu tests/test_gpu_debug_asserts.py 2>&1 | tail -5 > gpurun_out/gpu13b.log
