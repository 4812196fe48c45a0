#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
cat > /tmp/tma_small.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np
import paper_1405_6162_b200 as lk
from paper_1405_6162_b200.kernels import random_binary_state
lk.cs_variant(lk.CS_TMA)
shape = lk.LatticeShape(*[int(v) for v in sys.argv[1].split("x")])
f0, g0 = random_binary_state(shape, np.random.default_rng(3))
with lk.BinaryFluid(shape, mode=lk.MODE_FAST, use_graph=False) as sim:
    sim.load(f0, g0); sim.run(2); f1, g1 = sim.fields()
print("ok", float(f1.data.sum()))
PY
timeout 900 compute-sanitizer --tool memcheck python /tmp/tma_small.py 256x128x32 > gpurun_out/san_mem.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck python /tmp/tma_small.py 256x128x32 > gpurun_out/san_sync.txt 2>&1
for i in 1 2 3; do timeout 300 python /tmp/tma_small.py 256x256x256 >> gpurun_out/san_plain.txt 2>&1; done
for l in 0 1; do LTK_TMA_LOADER=$l timeout 600 python -m pytest tests/test_gpu_fluid.py tests/test_gpu_peer.py -x -q -m gpu -k "Tma or tma" -p no:cacheprovider >> gpurun_out/san_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/san_pytest.log; done
LTK_CS_VARIANT=1 timeout 300 python bench.py --mode fast --no-e2e --no-cpu-baseline > gpurun_out/san_bench.json 2> gpurun_out/san_bench.err
