#!/bin/bash
mkdir -p gpurun_out
HDG_MAX_GRID=4 timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_case.py C4 C2 > gpurun_out/racecheck_C4.log 2>&1; echo "rc=$?" >> gpurun_out/racecheck_C4.log
tail -6 gpurun_out/racecheck_C4.log
timeout 900 python bench.py --config C5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_C5_chunked.log 2>&1; echo "rc=$?" >> gpurun_out/bench_C5_chunked.log
tail -3 gpurun_out/bench_C5_chunked.log | cut -c1-1500
