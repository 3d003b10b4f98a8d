#!/bin/bash
# quick GPU check: parity tests (both condensation kernels) + condense/assemble/backsub times per config
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
HDG_CONDENSE_KERNEL=sweep timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_sweep.log
HDG_CONDENSE_KERNEL=panel timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_panel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_panel.log
for c in ${CONFIGS:-C1 C2 C3 C4}; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
true
