#!/bin/bash
# Full-step bench per force form (EXACT, tau 1), plus a launch list of the stress form.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for p in binary binary-stress passive; do
timeout 300 python bench.py --physics $p --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/bench_phys_$p.json 2>> gpurun_out/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -c 40 --csv --log-file gpurun_out/launches_stress.csv python bench.py --physics binary-stress --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_ncu.py launches gpurun_out/launches_stress.csv gpurun_out/launches_stress.json > /dev/null 2>&1
