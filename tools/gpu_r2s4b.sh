#!/bin/bash
# round 2, session 4: streaming (evict-first) hints on the factor / S stores and the GT input loads; the GT slabs
# as a persisting L2 window (HDG_GT_PERSIST=<MB>); parity of the sweep paths
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pivot_fullpath_gpu.py tests/test_parity_gpu.py -x -q -p no:cacheprovider > gpurun_out/s4b_pytest.log 2>&1; tail -2 gpurun_out/s4b_pytest.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], 'cond_ms %.3f step %.3f bs %.3f' % (d['condense_ms'], d['ms_per_step'], d['backsub_ms']), 'frac %.3f' % d['roofline']['frac'])"; }
for v in "X=1" "HDG_GT_PERSIST=40" "HDG_GT_PERSIST=80"; do
  n=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4b_C5s_$n.log 2>&1; show gpurun_out/s4b_C5s_$n.log
  grep HDG_GT_PERSIST gpurun_out/s4b_C5s_$n.log | head -1
done
for c in C4 C3; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4b_$c.log 2>&1; show gpurun_out/s4b_$c.log
done
