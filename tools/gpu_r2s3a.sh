#!/bin/bash
# session-3 first check: GPU suite + default bench on HEAD, C3 cycle traces (panel and sweep kernels)
O=gpurun_out/s3a; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_C4.jsonl 2> $O/bench_C4.err
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_C3.jsonl 2> $O/bench_C3.err
timeout 120 python tools/trace_condense.py --config C3 > $O/trace_C3_panel.txt 2>&1
HDG_CONDENSE_KERNEL=sweep timeout 120 python tools/trace_sweep.py --config C3 > $O/trace_C3_sweep.txt 2>&1
timeout 120 python tools/trace_sweep.py --config C4 > $O/trace_C4_sweep.txt 2>&1
