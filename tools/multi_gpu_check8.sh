#!/bin/bash
# 8-GPU parity + benches (run on an 8-GPU box): B toroidal, C = 4 toroidal x 2
# particle (fp64), D = 4 toroidal x 2 radial (fp32 state) at full size
N=8
run() { NCCL_DEBUG=WARN timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) "$@"; }
run tests/dist_parity.py --size T --mzetamax 16 2>&1 | grep -E "world|Error" | cut -c1-200
run tests/dist_parity.py --size A --nparts 1000000 2>&1 | grep -E "world|Error" | cut -c1-200
run tests/dist_parity.py --size A --nparts 1000000 --npartdom 2 2>&1 | grep -E "world|Error" | cut -c1-200
run tests/dist_parity.py --size A --nparts 1000000 --nradial 2 --precision 32 2>&1 | grep -E "world|Error" | cut -c1-200
NCCL_DEBUG=WARN timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus $N --steps 10 --warmup 3 --no-e2e > gpurun_out/bench8.log 2>&1
grep -oE "\"value\": [0-9.]+|\"ms_per_step\": [0-9.]+|\"phase_ms_per_step\": \{[^}]*\}" gpurun_out/bench8.log
tail -3 gpurun_out/bench8.log | grep -iE "error" | head -3
for cfg in "--size C --npartdom 2" "--size D --nradial 2 --precision 32"; do
  NCCL_DEBUG=WARN timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29900 + RANDOM % 90)) bench.py --gpus $N $cfg --steps 3 --warmup 3 --no-e2e --no-cpu \
      > gpurun_out/bench8_cfg.log 2>&1
  echo "$cfg"; grep -oE "\"value\": [0-9.]+|\"ms_per_step\": [0-9.]+" gpurun_out/bench8_cfg.log
done
