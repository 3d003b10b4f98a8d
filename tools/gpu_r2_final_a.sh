#!/bin/bash
# round-2 final evidence, part A: full GPU suite, smoke, default bench line (e2e + cpu_baseline), reference arm,
# launch list of the default bench, ncu --set full of the C4 sweep kernel
O=gpurun_out/r02; mkdir -p $O gpurun_out/ncu
nvidia-smi -L > $O/smi.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_default.jsonl 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.jsonl 2> $O/bench_reference.err
N=gpurun_out/ncu
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $N/plain_default.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $N/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $N/ncu_launches.log 2>&1
timeout 300 python tools/prof_case.py --config C4 --reps 2 > $N/plain_prof_case.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $N/sweep_C4 python tools/prof_case.py --config C4 --reps 2 > $N/ncu_sweep.log 2>&1
ls -la $O $N
