#!/bin/bash
# round 2, session 4: DMMA/DFMA pipe sharing microbenchmark; C3 on the 16-warp shared-memory sweep
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mix tools/micro/dmma_dfma_mix.cu && timeout 120 /tmp/mix > gpurun_out/mix.json 2>&1
cat gpurun_out/mix.json
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], 'cond_ms %.3f step %.3f' % (d['condense_ms'], d['ms_per_step']), d['roofline']['kernel'], 'frac %.3f' % d['roofline']['frac'])"; }
for v in "X=1" "HDG_CONDENSE_KERNEL=sweep" "HDG_CONDENSE_KERNEL=sweep HDG_SWEEP_WARPS=16"; do
  n=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4a_C3_$n.log 2>&1; show gpurun_out/s4a_C3_$n.log
done
env HDG_SWEEP_WARPS=16 timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4a_C4_w16.log 2>&1; show gpurun_out/s4a_C4_w16.log
timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4a_C4.log 2>&1; show gpurun_out/s4a_C4.log
