#!/bin/bash
# round 2, session 4: GT sweep discards the dead slab rows from L2 (HDG_DEBUG_MODE=16 switches it off)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pivot_fullpath_gpu.py tests/test_parity_gpu.py tests/test_fullsize_gpu.py -x -q -p no:cacheprovider > gpurun_out/s4c_pytest.log 2>&1; tail -2 gpurun_out/s4c_pytest.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f bs %.3f' % (d['condense_ms'], d['ms_per_step'], d['backsub_ms']), 'frac %.3f' % d['roofline']['frac'])"; }
for r in 1 2; do
for v in "X=1" "HDG_DEBUG_MODE=16"; do
  n=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4c_C5s_$n.log 2>&1; show gpurun_out/s4c_C5s_$n.log
done
done
timeout 300 python bench.py --config C5 --slab 0/8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"sweep_kernel<16" -c 4 --csv python bench.py --config C5 --slab 0/8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/s4c_ncu_gt.csv 2>&1
grep -E "dram__|gpu__time|lts__" gpurun_out/s4c_ncu_gt.csv | head -20
