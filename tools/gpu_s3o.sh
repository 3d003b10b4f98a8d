#!/bin/bash
# upd_part16 (predicated, hoisted partial trailing blocks) A/B within one binary (HDG_DEBUG_MODE=32 = old path)
O=gpurun_out/s3o; mkdir -p $O
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="timeout 200 python bench.py --config C4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
$B > $O/C4_new.jsonl 2>&1
HDG_DEBUG_MODE=32 $B > $O/C4_old.jsonl 2>&1
$B > $O/C4_new2.jsonl 2>&1
HDG_DEBUG_MODE=32 $B > $O/C4_old2.jsonl 2>&1
