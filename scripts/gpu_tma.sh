#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for l in 0 1; do LTK_TMA_LOADER=$l timeout 300 python -m pytest tests/test_gpu_fluid.py -x -q -m gpu -k "Tma" -p no:cacheprovider >> gpurun_out/tma_pytest.log 2>&1; done
echo "rc=$?" >> gpurun_out/tma_pytest.log
B="python bench.py --no-e2e --no-cpu-baseline"
LTK_CS_VARIANT=0 timeout 300 $B > gpurun_out/tma_reg.json 2>> gpurun_out/tma.err
for l in 0; do
LTK_TMA_LOADER=$l LTK_CS_VARIANT=1 timeout 300 $B > gpurun_out/tma_l$l.json 2>> gpurun_out/tma.err
done
LTK_TMA_LOADER=0 LTK_CS_VARIANT=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_cs_tma -s 1 -c 1 -o gpurun_out/full_cstma $B --steps 3 --warmup 3 > /dev/null 2>&1
