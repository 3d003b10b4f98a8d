#!/bin/bash
# iteration loop on the GPU: parity tests, sweep trace (C4), condense/assemble/backsub times per config
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python tools/trace_sweep.py --config C4 > gpurun_out/trace_sweep_C4.txt 2>&1
python tools/trace_sweep.py --config C3 --nr 32 --nt 64 > gpurun_out/trace_sweep_C3.txt 2>&1
for c in ${CONFIGS:-C3 C4}; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
true
