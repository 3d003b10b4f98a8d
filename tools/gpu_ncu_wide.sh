#!/bin/bash
mkdir -p gpurun_out/ncu
O=gpurun_out/ncu
export HDG_CONDENSE_KERNEL=wide
python tools/prof_case.py --config C3 --reps 1 > $O/plain_wide.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:warp_kernel -s 0 -c 1 -o $O/wide_C3 -f python tools/prof_case.py --config C3 --reps 1 > $O/ncu_wide.log 2>&1
tail -2 $O/ncu_wide.log
