#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_collision.py -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_coll.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_coll.log
run() {
timeout 300 python - <<'PY'
import sys, os; sys.path.insert(0, '.')
import paper_1405_6162_b200 as lk
tag = "NO_DIVC=%s MAXREG=%s" % (os.environ.get("LTK_NO_DIVC","0"), os.environ.get("LTK_MAXREG","0"))
for v in (1, 2):
    r = lk.benchmark_run("binary-collision", lk.LatticeShape(128,128,128), v, iterations=50, mode=lk.MODE_EXACT)
    print(tag, "vvl", v, round(r.sites_per_s/1e9, 3), "GLUPS", round(r.bandwidth_gb_s), "GB/s")
PY
}
( LTK_NO_DIVC=1 run; run; for m in 64 80 96; do LTK_MAXREG=$m run; LTK_NO_DIVC=1 LTK_MAXREG=$m run; done ) > gpurun_out/exp_exact.log 2>&1
