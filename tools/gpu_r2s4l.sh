#!/bin/bash
# streaming stores in GT mode only, all loads by __ldg: parity + C4 / p = 4 / C5 slab
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s4l_pytest.log 2>&1; tail -2 gpurun_out/s4l_pytest.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f bs %.3f' % (d['condense_ms'], d['ms_per_step'], d['backsub_ms']), 'frac %.3f' % d['roofline']['frac'])"; }
timeout 300 python bench.py --config C4 --degree 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4l_p4.log 2>&1; show gpurun_out/s4l_p4.log
timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4l_C5s.log 2>&1; show gpurun_out/s4l_C5s.log
timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4l_C4.log 2>&1; show gpurun_out/s4l_C4.log
timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4l_C4b.log 2>&1; show gpurun_out/s4l_C4b.log
