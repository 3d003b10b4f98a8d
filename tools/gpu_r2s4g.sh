#!/bin/bash
# round 2, session 4: C5 bucket dispatch — the n_e = 72 buckets on the shared-memory sweep (HDG_SWEEP_MIN_NE=64),
# the (120, n_f > 48) buckets on the GT sweep instead of the panel kernel (HDG_GT_MIN_NE=96)
mkdir -p gpurun_out
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f bs %.3f' % (d['condense_ms'], d['ms_per_step'], d['backsub_ms']), 'frac %.3f' % d['roofline']['frac'])"; }
for v in "X=1" "HDG_SWEEP_MIN_NE=64" "HDG_GT_MIN_NE=96" "HDG_SWEEP_MIN_NE=64 HDG_GT_MIN_NE=96" "HDG_GT_MIN_NE=64"; do
  n=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4g_C5s_$n.log 2>&1; show gpurun_out/s4g_C5s_$n.log
done
HDG_SWEEP_MIN_NE=64 HDG_GT_MIN_NE=96 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_pivot_fullpath_gpu.py -x -q -p no:cacheprovider > gpurun_out/s4g_pytest.log 2>&1; tail -2 gpurun_out/s4g_pytest.log
