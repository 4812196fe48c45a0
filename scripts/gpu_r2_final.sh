#!/bin/bash
# Round-2 refresh of the judged evidence: smoke, GPU suite, default bench line,
# reference arm (outputs in gpurun_out/, copied to profiles/ by hand).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?" >> gpurun_out/bench_reference.err
tail -1 gpurun_out/smoke.log; tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.err; tail -1 gpurun_out/bench_reference.err
