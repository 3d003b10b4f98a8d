#!/bin/bash
# warp-kernel iteration: parity (incl. full-path pivoting) + C1/C2 condense times, with/without the L2 prefetch
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_pivot_fullpath_gpu.py tests/test_fused_gpu.py tests/test_saved_solutions.py tests/test_recondense_gpu.py -q -x -p no:cacheprovider -rf > gpurun_out/pytest_c2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c2.log; tail -2 gpurun_out/pytest_c2.log
for m in 0; do for c in C1 C2; do HDG_DEBUG_MODE=$m timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('mode $m $c', {k: round(d[k],4) for k in ('ms_per_step','condense_ms','assemble_ms','backsub_ms')})"; done; done
