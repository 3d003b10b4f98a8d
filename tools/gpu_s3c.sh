#!/bin/bash
O=gpurun_out/s3c; mkdir -p $O
./tools/micro/slots > $O/slots.txt 2>&1
B="timeout 300 python bench.py --no-e2e --no-cpu-baseline"
HDG_SWEEP_ONE=1 HDG_CONDENSE_KERNEL=sweep $B --config C3 --steps 5 --warmup 3 > $O/C3_sweep_one.jsonl 2>&1
HDG_SWEEP_ONE=1 HDG_CONDENSE_KERNEL=sweep timeout 120 python tools/trace_sweep.py --config C3 > $O/trace_C3_sweep_one.txt 2>&1
