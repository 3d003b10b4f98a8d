#!/bin/bash
# round 2, session 4 evidence on the committed kernels: GPU suite + smoke, every bench line, the C4 launch list,
# ncu --set full of the C4 sweep kernel and of the C5 GT sweep (n_e = 252 bucket)
O=gpurun_out/s4f; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
bash tools/gpu_r2_evidence.sh > $O/evidence_summary.txt 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain_default.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 300 python tools/prof_case.py --config C4 --reps 2 > $O/plain_prof_case.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $O/sweep_C4 -f python tools/prof_case.py --config C4 --reps 2 > $O/ncu_sweep.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"sweep_kernel<16" -c 2 -o $O/gt_C5 -f python bench.py --config C5 --slab 0/8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_gt.log 2>&1
ls -la $O | tail -8
