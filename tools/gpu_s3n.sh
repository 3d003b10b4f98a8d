#!/bin/bash
# deferred [S|g] (issued in the next panel's TRSM phase): parity + C4 time + trace
O=gpurun_out/s3n; mkdir -p $O
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
HDG_CONDENSE_KERNEL=sweep timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "parity or pivot or fused or recondense or saved" > $O/pytest_sweep.log 2>&1; echo "rc=$?" >> $O/pytest_sweep.log
timeout 200 python bench.py --config C4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/C4.jsonl 2>&1
timeout 60 python tools/trace_sweep.py --config C4 > $O/trace_C4.txt 2>&1
timeout 200 python bench.py --config C5 --slab 0/8 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $O/C5slab.jsonl 2>&1
