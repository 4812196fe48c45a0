#!/bin/bash
# A/B of env configurations on the default bench line; usage: gpu_ab.sh "ENV=.. ENV2=.." "ENV=.." ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.txt
for cfg in "$@"; do
  for rep in 1 2; do
    echo "== $cfg" >> gpurun_out/ab.txt
    env $cfg timeout 120 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-config1 ${BENCH_ARGS} >> gpurun_out/ab.txt 2>&1
  done
done
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log; fi
