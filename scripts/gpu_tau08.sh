#!/bin/bash
# ncu --set full of k_collide_stream at tau = 0.8 (EXACT, every division live), summarised.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python bench.py --tau 0.8 --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/bench_tau08.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --tau 0.8 --mode fast --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/bench_tau08_fast.json 2>> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide_stream -s 3 -c 1 -o gpurun_out/prof_cs_tau08 python bench.py --tau 0.8 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_ncu.py report gpurun_out/prof_cs_tau08.ncu-rep gpurun_out/ncu_cs_tau08.json > /dev/null 2>&1
ncu -i gpurun_out/prof_cs_tau08.ncu-rep --page details --csv > gpurun_out/ncu_cs_tau08_details.csv 2>/dev/null
rm -f gpurun_out/prof_cs_tau08.ncu-rep
