#!/bin/bash
# Full GPU suite (row-blocked default), k_mu_blk min-blocks A/B, the 2-rank
# cross-process bench and the strong 512^3 line.  Run under gpurun.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
for M in 0 5 6; do
LTK_MU_MINB=$M timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/bench_minb${M}_$r.json 2>> gpurun_out/bench.err
done
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline --shape 128x128x64 > gpurun_out/p2_bench.json 2> gpurun_out/p2_bench.err
echo "rc=$?" >> gpurun_out/p2_bench.err
timeout 600 python bench.py --scaling strong --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_strong512.json 2>> gpurun_out/bench.err
