T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512"
$T bench.py --gpus 2 --size D --nradial 2 --mzetamax 16 --precision 32 --steps 3 --warmup 2 --no-e2e > gpurun_out/b11_D_rad2.json 2> gpurun_out/b11_D_rad2.err
$T bench.py --gpus 2 --size D --mzetamax 16 --precision 32 --steps 3 --warmup 2 --no-e2e > gpurun_out/b11_D_tor2.json 2> gpurun_out/b11_D_tor2.err
$T bench.py --gpus 2 --size C --npartdom 2 --mzetamax 16 --steps 3 --warmup 2 --no-e2e > gpurun_out/b11_C_part2.json 2> gpurun_out/b11_C_part2.err
