#!/bin/bash
# one full ncu capture of the C2 warp-per-element condensation kernel
mkdir -p gpurun_out/ncu
O=gpurun_out/ncu
python tools/prof_case.py --config C2 --reps 2 > $O/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:warp_kernel -s 1 -c 1 -o $O/warp_C2 python tools/prof_case.py --config C2 --reps 2 > $O/ncu_c2.log 2>&1
tail -3 $O/ncu_c2.log; ls -la $O | grep C2
