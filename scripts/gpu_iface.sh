#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
H="timeout 600 python scripts/exp_interface_hist.py 4x4x64 20000 2000"
$H -0.00625 0.00625 0.004 1.0 1.0 1.0 > gpurun_out/h_weak.json 2>>gpurun_out/h.err
$H -0.00625 0.00625 0.016 1.0 1.0 1.0 > gpurun_out/h_weakwide.json 2>>gpurun_out/h.err
$H -0.0625 0.0625 0.04 1.0 1.0 1.0 > gpurun_out/h_strong.json 2>>gpurun_out/h.err
$H -0.0625 0.0625 0.04 1.0 3.0 1.0 > gpurun_out/h_strong_visc.json 2>>gpurun_out/h.err
$H -0.0625 0.0625 0.04 0.0 1.0 1.0 > gpurun_out/h_strong_g0.json 2>>gpurun_out/h.err
