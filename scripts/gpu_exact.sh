#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_collision.py -x -q -m gpu -k "ExactDivision" -p no:cacheprovider > gpurun_out/exact_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/exact_pytest.log
timeout 300 python scripts/exp_tau.py > gpurun_out/exact_tau.txt 2>&1
timeout 300 python bench.py --mode exact --tau 0.8 --no-e2e --no-cpu-baseline > gpurun_out/exact_tau08.json 2>> gpurun_out/exact.err
timeout 300 python bench.py --mode fast --tau 0.8 --no-e2e --no-cpu-baseline > gpurun_out/fast_tau08.json 2>> gpurun_out/exact.err
