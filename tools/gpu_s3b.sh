#!/bin/bash
# SMSP role rotation A/B for the 2-CTA sweep (C3 forced to the sweep kernel); C4 control
O=gpurun_out/s3b; mkdir -p $O
B="timeout 300 python bench.py --no-e2e --no-cpu-baseline"
HDG_CONDENSE_KERNEL=sweep timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "parity or pivot" > $O/pytest_sweep.log 2>&1; echo "rc=$?" >> $O/pytest_sweep.log
HDG_CONDENSE_KERNEL=sweep $B --config C3 --steps 5 --warmup 3 > $O/C3_sweep_rot.jsonl 2>&1
HDG_CONDENSE_KERNEL=sweep HDG_DEBUG_MODE=4 $B --config C3 --steps 5 --warmup 3 > $O/C3_sweep_norot.jsonl 2>&1
$B --config C3 --steps 5 --warmup 3 > $O/C3_panel.jsonl 2>&1
HDG_CONDENSE_KERNEL=sweep timeout 120 python tools/trace_sweep.py --config C3 > $O/trace_C3_sweep_rot.txt 2>&1
