#!/bin/bash
# row-tile kernel bring-up: parity with the oracle (forced via HDG_CONDENSE_KERNEL=rows), then timings vs. default
mkdir -p gpurun_out
export HDG_CONDENSE_KERNEL=rows
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "uniform_configs_reduced_mesh and (C3 or C4)" > gpurun_out/rows_parity.log 2>&1; echo "rc=$?" >> gpurun_out/rows_parity.log
tail -3 gpurun_out/rows_parity.log
if grep -q "rc=0" gpurun_out/rows_parity.log; then
  timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_pivot_fullpath_gpu.py -q -p no:cacheprovider -k "not panel and not sweep and not c2_sized and not two_rank and not exchange" > gpurun_out/rows_parity2.log 2>&1; echo "rc=$?" >> gpurun_out/rows_parity2.log
  tail -5 gpurun_out/rows_parity2.log
  for c in C4 C3; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_rows_$c.log 2>&1; tail -1 gpurun_out/bench_rows_$c.log | cut -c1-400; done
fi
unset HDG_CONDENSE_KERNEL
for c in C4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_def_$c.log 2>&1; tail -1 gpurun_out/bench_def_$c.log | cut -c1-400; done
