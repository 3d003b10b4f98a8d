#!/bin/bash
# CREG (C_e row tiles in registers) A/B in one binary (HDG_DEBUG_MODE=64 = off)
O=gpurun_out/s3r; mkdir -p $O
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="timeout 200 python bench.py --config C4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
$B > $O/C4_creg.jsonl 2>&1
HDG_DEBUG_MODE=64 $B > $O/C4_off.jsonl 2>&1
$B > $O/C4_creg2.jsonl 2>&1
timeout 60 python tools/trace_sweep.py --config C4 > $O/trace_C4.txt 2>&1
