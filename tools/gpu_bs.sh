#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_pivot_fullpath_gpu.py -q -x -p no:cacheprovider -rf > gpurun_out/pytest_bs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bs.log; tail -2 gpurun_out/pytest_bs.log
for c in C4 C3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('$c', {k: round(d[k],3) for k in ('ms_per_step','condense_ms','assemble_ms','backsub_ms','backsub_hbm_gbs')})"; done
timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C5s.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_C5s.log').read().strip().splitlines()[-1]); print('C5s', {k: round(d[k],3) for k in ('ms_per_step','condense_ms','assemble_ms','backsub_ms','backsub_hbm_gbs')})"
