#!/bin/bash
# Round-end evidence: full GPU tests, every config's bench line, the default bench line (with e2e and
# cpu_baseline), the reference arm, the ncu launch list of the default bench and one full capture per hot kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
for c in C1 C2 C3 C4 C5; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
for c in C3 C4; do timeout 400 python bench.py --path adjoint --config $c --steps 5 --warmup 3 > gpurun_out/bench_adjoint_$c.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/sweep_full_C4 -f python tools/prof_case.py --config C4 --reps 2 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:condense_kernel -s 1 -c 1 -o gpurun_out/panel_full_C3 -f python tools/prof_case.py --config C3 --reps 2 > gpurun_out/ncu_full_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:backsub_kernel -s 1 -c 1 -o gpurun_out/backsub_full_C4 -f python tools/prof_case.py --config C4 --reps 2 > gpurun_out/ncu_full_bs.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sweep_kernel|condense_kernel|backsub|assemble" -c 120 --csv --log-file gpurun_out/launches_C5.csv python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_C5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o gpurun_out/sweep_gt_C5 -f python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_c5.log 2>&1
true
