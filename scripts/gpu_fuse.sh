#!/bin/bash
# Fused-step check: GPU tests of the fluid path, then a fused bench sweep.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fluid.py tests/test_gpu_peer.py -x -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_fuse.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_fuse.log
B="python bench.py --no-e2e --no-cpu-baseline"
for h in ${HINTS:-0 2 3}; do for lag in ${LAGS:-0 1 2 4}; do
  LTK_FUSE_HINT=$h timeout 300 $B --fuse --fuse-lag $lag > gpurun_out/bench_fuse_h${h}_lag$lag.json 2>> gpurun_out/bench_fuse.err
done; done
timeout 300 $B > gpurun_out/bench_nofuse.json 2>> gpurun_out/bench_fuse.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_fuse.csv $B --steps 3 --warmup 3 > /dev/null 2>&1
echo done >> gpurun_out/bench_fuse.err
