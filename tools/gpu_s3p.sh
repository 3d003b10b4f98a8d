#!/bin/bash
# PAIR trailing updates (k = 32 at odd panels): parity, C4 time, trace, C5 slab
O=gpurun_out/s3p; mkdir -p $O
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
$B --config C4 > $O/C4.jsonl 2>&1
$B --config C4 > $O/C4b.jsonl 2>&1
timeout 60 python tools/trace_sweep.py --config C4 > $O/trace_C4.txt 2>&1
$B --config C5 --slab 0/8 > $O/C5slab.jsonl 2>&1
