#!/bin/bash
mkdir -p gpurun_out
export HDG_CONDENSE_KERNEL=rows
timeout 300 python -m pytest tests/test_parity_gpu.py tests/test_pivot_fullpath_gpu.py -q -x -p no:cacheprovider -k "(uniform_configs_reduced_mesh and (C3 or C4)) or hp_config or test_pivot_forcing or c4_sized and default or c3_sized and default or hp_mesh" > gpurun_out/rows_parity.log 2>&1; echo "rc=$?" >> gpurun_out/rows_parity.log
tail -2 gpurun_out/rows_parity.log
for D in 1 2 3; do
  export HDG_ROWS_DELAY=$D
  timeout 300 python tools/trace_rows.py --config C3 --nr 64 --nt 64 --show 60 > gpurun_out/trace_rows_C3_d$D.txt 2>&1
  echo "D=$D"; tail -2 gpurun_out/trace_rows_C3_d$D.txt | head -1
  timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_rows_C3_d$D.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_rows_C3_d$D.log').read().strip().splitlines()[-1]); print('C3', 'condense_ms', round(d['condense_ms'],2), 'frac', round(d['roofline']['frac'],3))"
done
