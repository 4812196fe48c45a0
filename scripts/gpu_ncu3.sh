#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide_stream -s 1 -c 1 -o gpurun_out/full_cs $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_phi -s 3 -c 1 -o gpurun_out/full_phi $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cs_phi -s 1 -c 1 -o gpurun_out/full_csphi $B --fuse > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
