#!/bin/bash
# Round-2 GPU session b: physics pins, bench (configs[1] sub-record, reference
# numba CPU), the self-spawning multi-rank bench on the one GPU, reference arm.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_physics.py tests/test_gpu_bench.py -q -s -m gpu --timeout 500 -p no:cacheprovider > gpurun_out/pytest_physics.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_physics.log
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
timeout 300 python bench.py --gpus 4 --shape 64x64x64 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_spawn4.json 2> gpurun_out/bench_spawn4.err; echo "rc=$?" >> gpurun_out/bench_spawn4.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_collide --csv --log-file gpurun_out/ncu_collide128.csv python -c "
import sys; sys.path.insert(0,'.')
import paper_1405_6162_b200 as lk
from paper_1405_6162_b200.bench import benchmark_run
for v in (1,2,4,8):
    benchmark_run('binary-collision', lk.LatticeShape(128,128,128), v, iterations=3, mode=lk.MODE_EXACT)
" > gpurun_out/ncu_collide128.out 2>&1
