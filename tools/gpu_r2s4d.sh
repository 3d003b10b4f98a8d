#!/bin/bash
# round 2, session 4: full GPU suite + smoke on the streaming-store / L2-discard build; C3 panel-kernel shapes
mkdir -p gpurun_out
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f bs %.3f' % (d['condense_ms'], d['ms_per_step'], d['backsub_ms']), 'frac %.3f' % d['roofline']['frac'])"; }
for v in "X=1" "HDG_PANEL_CFG=128x3" "HDG_PANEL_CFG=256x1" "HDG_PANEL_CFG=256x2"; do
  n=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4d_C3_$n.log 2>&1; show gpurun_out/s4d_C3_$n.log
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s4d_pytest_gpu.log 2>&1; tail -3 gpurun_out/s4d_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4d_smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/s4d_smoke.log
