#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python scripts/debug_vvl2.py > gpurun_out/debug_vvl2.log 2>&1
# collision-only VVL sweep at 128^3 (configs[1]), EXACT and FAST
timeout 300 python - > gpurun_out/sweep128.log 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import paper_1405_6162_b200 as lk
for mode in (lk.MODE_EXACT, lk.MODE_FAST):
    for tpb in (128, 256):
        rows = lk.run_sweep("binary-collision", lk.LatticeShape(128, 128, 128), [1, 2, 4, 8, 16], [1], ["cuda"], iterations=50, tpb=tpb, mode=mode)
        print("mode", mode, "tpb", tpb)
        print(lk.emit_table(rows), lk.report_best(rows))
PY
for m in exact fast; do for v in 1 2; do
timeout 300 python bench.py --mode $m --vvl $v --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_${m}_v${v}.json 2>> gpurun_out/bench_explore.err
done; done
# ncu: launch list + one full capture of the collide-stream kernel (exact and fast)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_collide_stream -s 2 -c 1 -o gpurun_out/prof_cs_exact python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --shape 256x256x128 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_collide_stream -s 2 -c 1 -o gpurun_out/prof_cs_fast python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --mode fast --shape 256x256x128 > /dev/null 2>&1
ls -la gpurun_out
