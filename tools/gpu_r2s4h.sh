#!/bin/bash
# round 2, session 4: n_e = 72 buckets on the shared-memory sweep by default — GPU suite (incl. the new NS p = 2
# full-depth pivot test), C5 slab and whole mesh
O=gpurun_out/s4h; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'][:12], 'cond_ms %.3f step %.3f bs %.3f' % (d['condense_ms'], d['ms_per_step'], d['backsub_ms']), 'frac %.3f' % d['roofline']['frac'])"; }
timeout 300 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/C5s.log 2>&1; show $O/C5s.log
timeout 600 python bench.py --config C5 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $O/C5w.log 2>&1; show $O/C5w.log
