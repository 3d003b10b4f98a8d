#!/bin/bash
# GT sweep on the uniform p = 4 mesh (C4 mesh, n_e = 180): streaming input loads (debug 64 off) and the L2 discard
# (debug 16 off) A/B
mkdir -p gpurun_out
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f bs %.3f' % (d['condense_ms'], d['ms_per_step'], d['backsub_ms']), 'frac %.3f' % d['roofline']['frac'])"; }
for r in 1 2; do
for v in "X=1" "HDG_DEBUG_MODE=16" "HDG_DEBUG_MODE=64" "HDG_DEBUG_MODE=80"; do
  n=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --config C4 --degree 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4j_p4_$n.log 2>&1; show gpurun_out/s4j_p4_$n.log
done
done
for v in "X=1" "HDG_DEBUG_MODE=80"; do
  n=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4j_C5s_$n.log 2>&1; show gpurun_out/s4j_C5s_$n.log
done
