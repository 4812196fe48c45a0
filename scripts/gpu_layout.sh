#!/bin/bash
# Row-blocked vs SoA f/g layout: GPU tests, then alternating benches.  Run under gpurun.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
for L in soa row; do
timeout 300 python bench.py --layout $L --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/bench_${L}_exact_$r.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --layout $L --mode fast --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/bench_${L}_fast_$r.json 2>> gpurun_out/bench.err
done
done
for L in soa row; do
timeout 300 python bench.py --layout $L --shape 512x512x64 --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/bench_${L}_512.json 2>> gpurun_out/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_row.csv python bench.py --layout row --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_ncu.py launches gpurun_out/launches_row.csv gpurun_out/launches_row.json > /dev/null 2>&1
