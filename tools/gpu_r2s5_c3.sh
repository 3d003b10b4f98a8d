#!/bin/bash
# C3 on the sweep kernel (one CTA per SM through the grid cap) vs the panel kernel, after the session-5 sweep changes
O=gpurun_out/s5e; mkdir -p $O
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f' % (d['condense_ms'], d['ms_per_step']), 'frac %.3f' % d['roofline']['frac'])"; }
Q="--no-e2e --no-cpu-baseline"
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 $Q > $O/C3_panel.log 2>&1; show $O/C3_panel.log
HDG_SWEEP_MIN_NE=60 HDG_MAX_GRID=148 timeout 300 python bench.py --config C3 --steps 5 --warmup 3 $Q > $O/C3_sweep1.log 2>&1; show $O/C3_sweep1.log
for h in 10 18 24; do
HDG_DEBUG_MODE=$((h<<8)) HDG_SWEEP_MIN_NE=60 HDG_MAX_GRID=148 timeout 300 python bench.py --config C3 --steps 5 --warmup 3 $Q > $O/C3_sweep1_h$h.log 2>&1; echo hsel $h; show $O/C3_sweep1_h$h.log
done
HDG_SWEEP_MIN_NE=60 timeout 300 python bench.py --config C3 --steps 5 --warmup 3 $Q > $O/C3_sweep2.log 2>&1; show $O/C3_sweep2.log
