#!/bin/bash
# panel kernel phase B: one item per warp pass (default) vs two (debug 64) on C3 and the C5 slab
O=gpurun_out/s5p; mkdir -p $O
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f' % (d['condense_ms'], d['ms_per_step']), 'frac %.3f' % d['roofline']['frac'])"; }
Q="--no-e2e --no-cpu-baseline"
for m in 0 64; do
HDG_DEBUG_MODE=$m timeout 300 python bench.py --config C3 --steps 5 --warmup 3 $Q > $O/C3_m$m.log 2>&1; echo "mode $m"; show $O/C3_m$m.log
HDG_DEBUG_MODE=$m timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 $Q > $O/C5s_m$m.log 2>&1; show $O/C5s_m$m.log
HDG_DEBUG_MODE=$m timeout 300 python bench.py --config C4 --steps 5 --warmup 3 $Q > $O/C4_m$m.log 2>&1; show $O/C4_m$m.log
done
