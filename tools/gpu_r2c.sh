#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_saved_solutions.py tests/test_recondense_gpu.py -q -p no:cacheprovider -rf > gpurun_out/pytest_saved.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_saved.log
tail -4 gpurun_out/pytest_saved.log
timeout 300 python bench.py --config C4 --path saved --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C4_saved.log 2>&1; tail -1 gpurun_out/bench_C4_saved.log | cut -c1-300
python -c "
import json; d=json.loads(open('gpurun_out/bench_C4_saved.log').read().strip().splitlines()[-1]); print({k: d[k] for k in ('condense_ms','save_solutions_ms','assemble_ms','backsub_ms','backsub_saved_bytes')})"
for c in C1 C2; do timeout 300 python bench.py --config $c --graph 100 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_${c}_graph.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_${c}_graph.log').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],4), d.get('cuda_graph'), round(d['condense_ms'],4))"; done
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['cpu_baseline'], d['e2e'])"
