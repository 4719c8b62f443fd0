#!/bin/bash
# Multi-GPU parity + bench sweep (run under gpurun --gpus N).  Usage: tools/multi_gpu_check.sh N
N=${1:-4}
run() {
    NCCL_DEBUG=WARN timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $((29500 + RANDOM % 400)) "$@" > gpurun_out/dist_last.log 2>&1
    rc=$?
    echo "rc=$rc $* :: $(grep -o '"ok": [a-z]*' gpurun_out/dist_last.log | head -1)"
    grep -h '^{' gpurun_out/dist_last.log >> gpurun_out/dist_parity_$N.jsonl
}
run tests/dist_parity.py --size T --mzetamax 8
run tests/dist_parity.py --size A --nparts 1000000
run tests/dist_parity.py --size T --mzetamax 8 --npartdom 2
run tests/dist_parity.py --size A --nparts 1000000 --npartdom 2
run tests/dist_parity.py --size T --mzetamax 8 --nradial 2
run tests/dist_parity.py --size A --nparts 1000000 --nradial 2
run tests/dist_parity.py --size A --nparts 1000000 --nradial 2 --precision 32
NCCL_DEBUG=WARN timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus $N --steps 5 --warmup 3 --no-e2e > gpurun_out/bench$N.log 2>&1
grep -oE "\"value\": [0-9.]+|\"ms_per_step\": [0-9.]+|\"phase_ms_per_step\": \{[^}]*\}" gpurun_out/bench$N.log
