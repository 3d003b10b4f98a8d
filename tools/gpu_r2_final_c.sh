#!/bin/bash
# round-2 final evidence (after the 128-byte factor records): ncu launch list + sweep capture first (traffic.json is
# refreshed from it before the bench lines), full GPU suite, smoke
O=gpurun_out/r02; N=gpurun_out/ncu; mkdir -p $O $N
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $N/plain_default.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $N/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $N/ncu_launches.log 2>&1
timeout 300 python tools/prof_case.py --config C4 --reps 2 > $N/plain_prof_case.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $N/sweep_C4 -f python tools/prof_case.py --config C4 --reps 2 > $N/ncu_sweep.log 2>&1
ls -la $O $N
