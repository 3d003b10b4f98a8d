#!/bin/bash
# row-tile kernel iteration: quick parity (forced), task timeline, C4/C3 timings
mkdir -p gpurun_out
export HDG_CONDENSE_KERNEL=rows
timeout 300 python -m pytest tests/test_parity_gpu.py tests/test_pivot_fullpath_gpu.py -q -x -p no:cacheprovider -k "(uniform_configs_reduced_mesh and (C3 or C4)) or hp_config or test_pivot_forcing or c4_sized and default or c3_sized and default or hp_mesh" > gpurun_out/rows_parity.log 2>&1; echo "rc=$?" >> gpurun_out/rows_parity.log
tail -2 gpurun_out/rows_parity.log
if grep -q "rc=0" gpurun_out/rows_parity.log; then
  timeout 300 python tools/trace_rows.py --config C4 --nr 32 --nt 64 --show 90 > gpurun_out/trace_rows_C4.txt 2>&1
  timeout 300 python tools/trace_rows.py --config C3 --nr 64 --nt 64 --show 60 > gpurun_out/trace_rows_C3.txt 2>&1
  tail -3 gpurun_out/trace_rows_C4.txt; tail -3 gpurun_out/trace_rows_C3.txt
  for c in C4 C3; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_rows_$c.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_rows_$c.log').read().strip().splitlines()[-1]); print('$c', 'condense_ms', round(d['condense_ms'],2), 'frac', round(d['roofline']['frac'],3), d['clocks'])"; done
fi
