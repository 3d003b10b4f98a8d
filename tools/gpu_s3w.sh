#!/bin/bash
# float block-row division adopted: parity, C4 time, C5 slab, ncu capture of the C4 sweep (traffic.json)
O=gpurun_out/s3w; mkdir -p $O
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
$B --config C4 > $O/C4.jsonl 2>&1
$B --config C4 > $O/C4b.jsonl 2>&1
$B --config C5 --slab 0/8 > $O/C5slab.jsonl 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain_default.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 300 python tools/prof_case.py --config C4 --reps 2 > $O/plain_prof_case.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $O/sweep_C4 -f python tools/prof_case.py --config C4 --reps 2 > $O/ncu_sweep.log 2>&1
