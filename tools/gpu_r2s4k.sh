#!/bin/bash
# streaming (st.global.cs) vs plain factor / S stores (libhdg_var.so = -DHDG_PLAIN_STORES), GT input loads by __ldg
mkdir -p gpurun_out
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f bs %.3f' % (d['condense_ms'], d['ms_per_step'], d['backsub_ms']), 'frac %.3f' % d['roofline']['frac'])"; }
for r in 1 2; do
for v in "X=1" "HDG_LIB_VARIANT=libhdg_var.so"; do
  n=$(echo $v | tr ' =.' '___')
  env $v timeout 300 python bench.py --config C4 --degree 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4k_p4_$n.log 2>&1; show gpurun_out/s4k_p4_$n.log
  env $v timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4k_C5s_$n.log 2>&1; show gpurun_out/s4k_C5s_$n.log
  env $v timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4k_C4_$n.log 2>&1; show gpurun_out/s4k_C4_$n.log
done
done
