#!/bin/bash
# sweep-kernel change check: parity (default + sweep forced everywhere, incl. pivot full path), C4/C5 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_pair.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pair.log; tail -2 gpurun_out/pytest_pair.log
HDG_CONDENSE_KERNEL=sweep timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_pivot_fullpath_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_pair_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pair_sweep.log; tail -2 gpurun_out/pytest_pair_sweep.log
for c in C4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('$c', {k: round(d[k],3) for k in ('ms_per_step','condense_ms')}, d['roofline']['frac'])"; done
timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C5s.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_C5s.log').read().strip().splitlines()[-1]); print('C5s', {k: round(d[k],3) for k in ('ms_per_step','condense_ms')})"
