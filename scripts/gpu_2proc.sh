#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_peer.py -x -q -m gpu -k two_process -p no:cacheprovider > gpurun_out/p2_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/p2_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline --shape 128x128x64 > gpurun_out/p2_bench.json 2> gpurun_out/p2_bench.err
echo "rc=$?" >> gpurun_out/p2_bench.err
