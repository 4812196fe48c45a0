#!/bin/bash
# compute-sanitizer over the engine (memcheck, racecheck, synccheck) on small lattices.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_engine.py > gpurun_out/san_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.txt
done
tail -3 gpurun_out/san_*.txt
