#!/bin/bash
# configs[1] collision-only VVL x TPB sweep at 128^3 (EXACT and FAST) through the
# latkit-compatible API, its ncu launch list, and the full step per mode x VVL.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python - > gpurun_out/sweep128.log 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import paper_1405_6162_b200 as lk
for mode in (lk.MODE_EXACT, lk.MODE_FAST):
    for tpb in (128, 256):
        rows = lk.run_sweep("binary-collision", lk.LatticeShape(128, 128, 128), [1, 2, 4, 8, 16], [1], ["cuda"], iterations=50, tpb=tpb, mode=mode)
        print("mode", mode, "tpb", tpb)
        print(lk.emit_table(rows), lk.report_best(rows))
PY
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_collision_128.csv python -c "
import sys; sys.path.insert(0,'.')
import paper_1405_6162_b200 as lk
for mode in (lk.MODE_EXACT, lk.MODE_FAST):
    for v in (1, 2, 4, 8):
        lk.benchmark_run('binary-collision', lk.LatticeShape(128,128,128), v, iterations=2, mode=mode)
" > /dev/null 2>&1
python scripts/summarize_ncu.py launches gpurun_out/launches_collision_128.csv gpurun_out/launches_collision_128.json > /dev/null 2>&1
for m in exact fast; do for v in 1 2; do
timeout 300 python bench.py --mode $m --vvl $v --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_${m}_v${v}.json 2>> gpurun_out/bench_explore.err
done; done
ls -la gpurun_out
