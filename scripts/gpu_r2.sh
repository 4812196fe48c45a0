#!/bin/bash
# Round-2 GPU session: physics pins (printed values), full GPU suite, one bench line.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_physics.py -q -s -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_physics.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_physics.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider --ignore=tests/test_gpu_physics.py > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
