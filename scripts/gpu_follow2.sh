#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for f in 0 1; do
LTK_FOLLOW=$f LTK_NCU_RANGE=1 timeout 600 ncu --replay-mode range --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --csv --log-file gpurun_out/ncu_range_f$f.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-config1 > gpurun_out/ncu_range_f$f.out 2>&1
done
