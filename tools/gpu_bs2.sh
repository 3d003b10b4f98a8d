#!/bin/bash
# back-substitution / adjoint change: parity + C4/C3/C5-slab back-sub and adjoint times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_pivot_fullpath_gpu.py tests/test_adjoint_gpu.py -q -x -p no:cacheprovider -rf > gpurun_out/pytest_bs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bs.log; tail -2 gpurun_out/pytest_bs.log
for c in C4 C3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('$c', {k: round(d[k],3) for k in ('ms_per_step','condense_ms','backsub_ms','backsub_hbm_gbs')})"; done
for c in C4 C3; do timeout 300 python bench.py --config $c --path adjoint --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_adj_$c.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_adj_$c.log').read().strip().splitlines()[-1]); print('adjoint $c', {k: round(d[k],3) for k in ('ms_per_step','adjoint_rhs_ms','backsub_adjoint_ms')})"; done
