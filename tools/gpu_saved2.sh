#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_saved_solutions.py tests/test_parity_gpu.py -q -x -p no:cacheprovider -rf > gpurun_out/pytest_saved2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_saved2.log; tail -3 gpurun_out/pytest_saved2.log
for c in C2 C3 C4; do for pth in primal saved; do timeout 300 python bench.py --config $c --path $pth --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_${c}_$pth.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_${c}_$pth.log').read().strip().splitlines()[-1]); print('$c $pth', {k: round(d[k],3) for k in ('ms_per_step','condense_ms','assemble_ms','backsub_ms')})"; done; done
