#!/bin/bash
# conflict-free accumulator row order in the panel kernel (C3, C5's n_e = 36 / 72 buckets)
O=gpurun_out/s3u; mkdir -p $O
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
$B --config C3 > $O/C3.jsonl 2>&1
$B --config C3 > $O/C3b.jsonl 2>&1
$B --config C5 --slab 0/8 > $O/C5slab.jsonl 2>&1
timeout 300 python tools/prof_case.py --config C3 --reps 2 > $O/plain_prof_case.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:condense_kernel -s 1 -c 1 -o $O/panel_C3 -f python tools/prof_case.py --config C3 --reps 2 > $O/ncu_panel.log 2>&1
