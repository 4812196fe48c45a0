#!/bin/bash
# div_rcp change: division self-test + full GPU suite, then tau 1 / 0.8 benches (EXACT, FAST).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for t in 1.0 0.8; do for m in exact fast; do
timeout 300 python bench.py --tau $t --mode $m --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/bench_tau${t}_$m.json 2>> gpurun_out/bench.err
done; done
timeout 300 python scripts/exp_tau.py > gpurun_out/collision_tau.txt 2>&1
