#!/bin/bash
# Round-2 full check: smoke, GPU tests, bench (default + reference arm),
# launch list and one ncu --set full capture per hot kernel.  Run under gpurun.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_exact.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-config1 > /dev/null 2>&1
for k in k_collide_stream k_phi k_mu_tile; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_$k python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-config1 > /dev/null 2>&1
python scripts/summarize_ncu.py report gpurun_out/prof_$k.ncu-rep gpurun_out/ncu_$k.json > /dev/null 2>&1
done
python scripts/summarize_ncu.py launches gpurun_out/launches_exact.csv gpurun_out/launches_exact.json > /dev/null 2>&1
rm -f gpurun_out/prof_k_phi.ncu-rep gpurun_out/prof_k_mu_tile.ncu-rep
ls -la gpurun_out
