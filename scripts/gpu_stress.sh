#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fluid.py tests/test_gpu_peer.py -x -q -m gpu -p no:cacheprovider > gpurun_out/stress_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/stress_pytest.log
H="timeout 600 python scripts/exp_interface_hist.py 4x4x64 20000 4000"
$H -0.0625 0.0625 0.04 1.0 1.0 1.0 > gpurun_out/hs_strong_pot.json 2>>gpurun_out/hs.err
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/stress_bench_default.json 2>>gpurun_out/hs.err
$H -0.0625 0.0625 0.04 1.0 1.0 1.0 binary-stress > gpurun_out/hs_strong_stress.json 2>>gpurun_out/hs.err
$H -0.00625 0.00625 0.036 1.0 1.0 1.0 binary-stress > gpurun_out/hs_wide_stress.json 2>>gpurun_out/hs.err
timeout 300 python bench.py --physics binary-stress --no-e2e --no-cpu-baseline > gpurun_out/stress_bench.json 2>>gpurun_out/hs.err
