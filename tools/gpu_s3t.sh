#!/bin/bash
# conflict-free accumulator row order (srow) in the sweep kernel's shared-memory updates
O=gpurun_out/s3t; mkdir -p $O
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
$B --config C4 > $O/C4.jsonl 2>&1
$B --config C4 > $O/C4b.jsonl 2>&1
$B --config C5 --slab 0/8 > $O/C5slab.jsonl 2>&1
HDG_CONDENSE_KERNEL=sweep HDG_SWEEP_ONE=1 $B --config C3 > $O/C3sweep.jsonl 2>&1
timeout 60 python tools/trace_sweep.py --config C4 > $O/trace_C4.txt 2>&1
timeout 300 python tools/prof_case.py --config C4 --reps 2 > $O/plain_prof_case.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $O/sweep_C4 -f python tools/prof_case.py --config C4 --reps 2 > $O/ncu_sweep.log 2>&1
