#!/bin/bash
# full GPU suite + the bench lines a sweep-kernel change can move (C4, C5 slab, C4 mesh at p = 4, C3)
O=gpurun_out/s5c; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f' % (d['condense_ms'], d['ms_per_step']), 'frac %.3f' % d['roofline']['frac'])"; }
Q="--no-e2e --no-cpu-baseline"
timeout 300 python bench.py --config C4 --steps 8 --warmup 3 $Q > $O/C4.log 2>&1; show $O/C4.log
timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 $Q > $O/C5s.log 2>&1; show $O/C5s.log
HDG_DEBUG_MODE=256 timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 $Q > $O/C5s_old.log 2>&1; show $O/C5s_old.log
for h in 12 13 15 16; do
  HDG_DEBUG_MODE=$((h << 8)) timeout 300 python bench.py --config C4 --steps 8 --warmup 3 $Q > $O/C4_h$h.log 2>&1; echo "hsel $h"; show $O/C4_h$h.log
done
