#!/bin/bash
# helper takes TRSM jobs in the first 2/3 panels (HDG_DEBUG_MODE bit 128 = off) and the float block-row division
# (bit 256 = integer): A/B within one binary
O=gpurun_out/s3v; mkdir -p $O
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="timeout 200 python bench.py --config C4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for m in 0 128 256 384 0 128 256 384; do HDG_DEBUG_MODE=$m $B > $O/C4_m$m.$RANDOM.jsonl 2>&1; done
