#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -m paper_1405_6162_b200.cli --kernel binary-collision --shape 128x128x128 --vvl 1,2,4,8,16 --iters 50 --mode exact > gpurun_out/cli_exact.txt 2>&1
timeout 300 python -m paper_1405_6162_b200.cli --kernel binary-collision --shape 128x128x128 --vvl 1,2,4,8,16 --iters 50 --mode fast > gpurun_out/cli_fast.txt 2>&1
timeout 300 python -m paper_1405_6162_b200.cli --kernel binary-fluid --shape 256x256x256 --vvl 1,2 --iters 20 --mode exact > gpurun_out/cli_fluid_exact.txt 2>&1
for m in exact fast; do
timeout 300 python bench.py --mode $m --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_$m.json 2>> gpurun_out/bench.err
done
