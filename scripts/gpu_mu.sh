#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for c in 0 1 2 3 4; do
LTK_MUCOL=$c timeout 600 python -m pytest tests/test_gpu_fluid.py -x -q -m gpu -k "Stencil or exact_bitwise" -p no:cacheprovider > gpurun_out/mu_pytest_$c.log 2>&1
echo "rc=$?" >> gpurun_out/mu_pytest_$c.log
LTK_MUCOL=$c timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/mu_bench_$c.json 2>> gpurun_out/mu_bench.err
done
