#!/bin/bash
O=gpurun_out/s3d; mkdir -p $O
./tools/micro/dmma_lat > $O/dmma_lat.txt 2>&1
B="timeout 300 python bench.py --no-e2e --no-cpu-baseline"
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "parity or pivot or fused" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
$B --config C4 --steps 10 --warmup 3 > $O/C4_rowmap.jsonl 2>&1
HDG_DEBUG_MODE=8 $B --config C4 --steps 10 --warmup 3 > $O/C4_rr.jsonl 2>&1
$B --config C4 --steps 10 --warmup 3 > $O/C4_rowmap2.jsonl 2>&1
timeout 120 python tools/trace_sweep.py --config C4 > $O/trace_C4.txt 2>&1
