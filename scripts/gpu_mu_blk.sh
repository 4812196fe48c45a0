#!/bin/bash
# k_mu_blk variants (batched centre loads; neighbour handling NB) vs k_mu_col:
# parity under the GPU tests, then alternating benches.  Run under gpurun.
# LTK_MU_BLK: 0 k_mu_col, 8 <8,0>, 9 <8,1> (next-plane neighbours prefetched),
# 10 <8,2> (outer y rows batched), 4 <4,1>
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for B in 9 10 4; do
LTK_MU_BLK=$B timeout 900 python -m pytest tests/test_gpu_fluid.py -q -m gpu --timeout 600 -p no:cacheprovider -x -k "Stencil or Stress or FullStep or RowLayout" > gpurun_out/pytest_mu_blk$B.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mu_blk$B.log
done
for r in 1 2; do
for B in 0 8 9 10 4; do
LTK_MU_BLK=$B timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/bench_mublk${B}_$r.json 2>> gpurun_out/bench.err
done
done
for B in 8 9 10 4; do
LTK_MU_BLK=$B timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_mu -c 4 --csv --log-file gpurun_out/mu_blk$B.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
timeout 300 python -m pytest tests/test_gpu_fluid.py -q -m gpu -k RowLayout -p no:cacheprovider > gpurun_out/pytest_row.log 2>&1
LTK_LAYOUT=0 timeout 300 python -m pytest tests/test_gpu_fluid.py -q -m gpu -k RowLayout -p no:cacheprovider > gpurun_out/pytest_row_soa.log 2>&1
