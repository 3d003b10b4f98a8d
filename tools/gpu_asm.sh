#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_asm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_asm.log; tail -2 gpurun_out/pytest_asm.log
for c in C4 C3 C2; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('$c', {k: round(d[k],4) for k in ('ms_per_step','condense_ms','assemble_ms','backsub_ms')})"; done
for c in C4 C3; do timeout 300 python bench.py --config $c --path saved --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_sv_$c.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_sv_$c.log').read().strip().splitlines()[-1]); print('saved $c', {k: round(d[k],4) for k in ('ms_per_step','condense_ms','assemble_ms','backsub_ms')})"; done
timeout 300 python bench.py --config C4 --path adjoint --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_adj.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_adj.log').read().strip().splitlines()[-1]); print('adjoint C4', {k: round(d[k],4) for k in d if k.endswith('_ms') or k=='ms_per_step'})"
