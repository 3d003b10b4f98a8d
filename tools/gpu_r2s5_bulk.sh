#!/bin/bash
# panel kernel: factor rows by TMA bulk stores (debug bit 32: the warp copy loop as before): parity, then the A/B
O=gpurun_out/s5g; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f' % (d['condense_ms'], d['ms_per_step']), 'frac %.3f' % d['roofline']['frac'])"; }
Q="--no-e2e --no-cpu-baseline"
for m in 0 32 0 32; do
HDG_DEBUG_MODE=$m timeout 300 python bench.py --config C3 --steps 5 --warmup 3 $Q > $O/C3_m$m.log 2>&1; echo "mode $m"; show $O/C3_m$m.log
done
for m in 0 32; do
HDG_DEBUG_MODE=$m timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 $Q > $O/C5s_m$m.log 2>&1; echo "mode $m"; show $O/C5s_m$m.log
done
