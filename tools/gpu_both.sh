#!/bin/bash
# condense times of both kernels on every config
mkdir -p gpurun_out
for c in ${CONFIGS:-C1 C2 C3 C4}; do
  HDG_CONDENSE_KERNEL=sweep timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_sweep_$c.log 2>&1
  HDG_CONDENSE_KERNEL=panel timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_panel_$c.log 2>&1
done
true
