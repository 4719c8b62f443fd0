set -x
python paper_1510_05546_b200/_build.py -DGTCP_DEP_CARRY --out=$PWD/paper_1510_05546_b200/_lib/libgtcp_carry.so > /dev/null
GTCP_LIB_PATH=$PWD/paper_1510_05546_b200/_lib/libgtcp_carry.so python -m pytest -q -m gpu tests/test_gpu_parity.py -k "charge or step_parity_T" 2>&1 | tail -3 > gpurun_out/carry_parity.log
python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/b3_default.json 2>&1
GTCP_LIB_PATH=$PWD/paper_1510_05546_b200/_lib/libgtcp_carry.so python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/b3_carry.json 2>&1
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_deposit_tiled -s 2 -c 1 -o gpurun_out/dep_r02a python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu3.log 2>&1
