#!/bin/bash
# Full round check: smoke, GPU tests, bench (default + exact + reference arm),
# launch list and one ncu --set full capture per hot kernel.  Run under gpurun.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --mode exact --no-e2e --no-cpu-baseline > gpurun_out/bench_exact.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_fast.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_exact.csv python bench.py --mode exact --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# one --set full capture per hot kernel, summarised on the box (the reports are
# large; only the dominant kernel's report is kept for source-level reading)
for k in k_collide_stream k_phi k_mu_lds; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_$k python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_ncu.py report gpurun_out/prof_$k.ncu-rep gpurun_out/ncu_$k.json > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 2 -c 1 -o gpurun_out/prof_k_collide_128 python -c "
import sys; sys.path.insert(0,'.')
import paper_1405_6162_b200 as lk
lk.benchmark_run('binary-collision', lk.LatticeShape(128,128,128), 1, iterations=3, mode=1)
" > /dev/null 2>&1
python scripts/summarize_ncu.py report gpurun_out/prof_k_collide_128.ncu-rep gpurun_out/ncu_k_collide_128.json > /dev/null 2>&1
python scripts/summarize_ncu.py launches gpurun_out/launches_fast.csv gpurun_out/launches_fast.json > /dev/null 2>&1
python scripts/summarize_ncu.py launches gpurun_out/launches_exact.csv gpurun_out/launches_exact.json > /dev/null 2>&1
rm -f gpurun_out/prof_k_phi.ncu-rep gpurun_out/prof_k_mu_lds.ncu-rep gpurun_out/prof_k_collide_128.ncu-rep
ls -la gpurun_out
