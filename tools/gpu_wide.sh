#!/bin/bash
# wide warp kernel (n_e <= 64): parity with it forced, C3 timing vs the panel kernel, C1/C2 unchanged
mkdir -p gpurun_out
HDG_CONDENSE_KERNEL=wide timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_pivot_fullpath_gpu.py tests/test_fullsize_gpu.py tests/test_recondense_gpu.py tests/test_saved_solutions.py tests/test_fused_gpu.py -q -x -p no:cacheprovider -rf > gpurun_out/pytest_wide.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_wide.log; tail -4 gpurun_out/pytest_wide.log
for k in panel wide; do HDG_CONDENSE_KERNEL=$k timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C3_$k.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_C3_$k.log').read().strip().splitlines()[-1]); print('$k C3', {k: round(d[k],3) for k in ('ms_per_step','condense_ms','assemble_ms','backsub_ms')})" || tail -3 gpurun_out/bench_C3_$k.log; done
for c in C1 C2; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('$c', {k: round(d[k],4) for k in ('ms_per_step','condense_ms')})"; done
