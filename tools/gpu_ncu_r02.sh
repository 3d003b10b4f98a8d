#!/bin/bash
# round-2 ncu evidence: the default bench's launch list, then one full capture each of the dominant kernels
mkdir -p gpurun_out/ncu
O=gpurun_out/ncu
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain_default.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1
python tools/prof_case.py --config C4 --reps 2 > $O/plain_prof_case.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $O/sweep_C4 python tools/prof_case.py --config C4 --reps 2 > $O/ncu_sweep.log 2>&1
HDG_CONDENSE_KERNEL=sweep python bench.py --config C4 --path saved --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/plain_saved.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"backsub_saved_kernel|save_kernel|backsub_kernel" -c 3 -o $O/saved_C4 python bench.py --config C4 --path saved --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_saved.log 2>&1
ls -la $O
