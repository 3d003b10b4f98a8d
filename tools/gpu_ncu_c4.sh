#!/bin/bash
# one full ncu capture of the C4 sweep kernel (roofline.traffic source)
mkdir -p gpurun_out/ncu
O=gpurun_out/ncu
python tools/prof_case.py --config C4 --reps 2 > $O/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $O/sweep_C4 -f python tools/prof_case.py --config C4 --reps 2 > $O/ncu_c4.log 2>&1
tail -2 $O/ncu_c4.log; ls -la $O | grep C4
