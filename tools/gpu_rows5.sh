#!/bin/bash
mkdir -p gpurun_out
export HDG_CONDENSE_KERNEL=rows
timeout 300 python -m pytest tests/test_recondense_gpu.py -q -x -p no:cacheprovider -k rows > gpurun_out/rows_shift.log 2>&1; echo "rc=$?" >> gpurun_out/rows_shift.log; tail -2 gpurun_out/rows_shift.log
for c in C3 C4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_rows_$c.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_rows_$c.log').read().strip().splitlines()[-1]); print('$c', 'condense_ms', round(d['condense_ms'],2), 'frac', round(d['roofline']['frac'],3))"; done
unset HDG_CONDENSE_KERNEL
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_C1.log 2>&1; tail -1 gpurun_out/bench_C1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['clocks'])"
