#!/bin/bash
# follow-mode A/B: bench lines, DRAM bytes of the whole step (ncu range replay), parity.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
rm -f gpurun_out/bench_follow.txt
B="timeout 120 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-config1"
for cfg in "LTK_FOLLOW=0" "LTK_FOLLOW=1" "LTK_FOLLOW=1 LTK_FOLLOW_DBG=1" "LTK_FOLLOW=1 LTK_FOLLOW_DBG=1 LTK_CS_CARVEOUT=-1" "LTK_FOLLOW=1 LTK_FOLLOW_DBG=2" "LTK_FOLLOW=1 LTK_FOLLOW_TPB=128 LTK_FOLLOW_DBG=1" ${EXTRA}; do
  echo "== $cfg" >> gpurun_out/bench_follow.txt
  env $cfg $B >> gpurun_out/bench_follow.txt 2>&1
done
LTK_FOLLOW=1 LTK_NCU_RANGE=1 timeout 600 ncu --replay-mode range --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/ncu_range_f1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-config1 > gpurun_out/ncu_range_f1.out 2>&1
if [ "$1" = "tests" ]; then
timeout 900 python -m pytest tests/test_gpu_fluid.py tests/test_gpu_physics.py -x -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_follow.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_follow.log
fi
