#!/bin/bash
# 11-warp shared-memory sweep (9 MMA workers, chain + helper alone on SMSP 3) vs 8 warps
O=gpurun_out/s3q; mkdir -p $O
HDG_SWEEP_WARPS=11 timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "parity or pivot or fused or recondense or saved or fullsize" > $O/pytest11.log 2>&1; echo "rc=$?" >> $O/pytest11.log
B="timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
HDG_SWEEP_WARPS=11 $B --config C4 > $O/C4_w11.jsonl 2>&1
$B --config C4 > $O/C4_w8.jsonl 2>&1
HDG_SWEEP_WARPS=11 $B --config C4 > $O/C4_w11b.jsonl 2>&1
HDG_SWEEP_WARPS=11 timeout 60 python tools/trace_sweep.py --config C4 > $O/trace_C4_w11.txt 2>&1
