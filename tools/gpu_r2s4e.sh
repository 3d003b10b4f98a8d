#!/bin/bash
# round 2, session 4: SMSP-aware chain/helper roles (two co-resident sweep CTAs keep both chains on SMSP 3);
# HDG_DEBUG_MODE=32 restores the fixed warp 7 / warp 3 roles
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pivot_fullpath_gpu.py tests/test_parity_gpu.py -x -q -p no:cacheprovider > gpurun_out/s4e_pytest.log 2>&1; tail -2 gpurun_out/s4e_pytest.log
HDG_CONDENSE_KERNEL=sweep timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -p no:cacheprovider -k "uniform or pivot or singular" > gpurun_out/s4e_pytest_sweep.log 2>&1; tail -2 gpurun_out/s4e_pytest_sweep.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f bs %.3f' % (d['condense_ms'], d['ms_per_step'], d['backsub_ms']), 'frac %.3f' % d['roofline']['frac'])"; }
for v in "HDG_CONDENSE_KERNEL=sweep" "HDG_CONDENSE_KERNEL=sweep HDG_DEBUG_MODE=32"; do
  n=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4e_C3_$n.log 2>&1; show gpurun_out/s4e_C3_$n.log
done
for c in C4 C2; do
for v in "X=1" "HDG_CONDENSE_KERNEL=sweep"; do
  n=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4e_${c}_$n.log 2>&1; show gpurun_out/s4e_${c}_$n.log
done
done
timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4e_C5s.log 2>&1; show gpurun_out/s4e_C5s.log
