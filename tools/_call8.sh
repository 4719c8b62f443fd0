python -m pytest -q -m gpu tests/test_gpu_parity.py -k 2gpu 2>&1 | tail -5 > gpurun_out/gpu8.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/b8_2gpu.json 2> gpurun_out/b8_2gpu.err
