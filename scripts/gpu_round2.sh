#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python - > gpurun_out/sweep128.log 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import paper_1405_6162_b200 as lk
for mode in (lk.MODE_EXACT, lk.MODE_FAST):
    for tpb in (128, 256):
        rows = lk.run_sweep("binary-collision", lk.LatticeShape(128, 128, 128), [1, 2, 4, 8, 16], [1], ["cuda"], iterations=50, tpb=tpb, mode=mode)
        print("mode", mode, "tpb", tpb)
        print(lk.emit_table(rows), lk.report_best(rows))
PY
timeout 600 python bench.py --steps 50 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_fast.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_collide -c 30 --csv --log-file gpurun_out/launches_coll128.csv python -c "
import sys; sys.path.insert(0,'.')
import paper_1405_6162_b200 as lk
for m in (0,1):
    for v in (1,2,4,8):
        lk.benchmark_run('binary-collision', lk.LatticeShape(128,128,128), v, iterations=2, mode=m)
" > /dev/null 2>&1
