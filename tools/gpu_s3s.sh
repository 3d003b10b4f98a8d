#!/bin/bash
# 128-byte factor records: GPU suite, C4 default / adjoint / saved timing, adjoint ncu (DRAM bytes), GT capture (C5)
O=gpurun_out/s3s; mkdir -p $O
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
$B --config C4 > $O/C4.jsonl 2>&1
$B --config C4 --path adjoint > $O/adjoint_C4.jsonl 2>&1
$B --config C3 --path adjoint > $O/adjoint_C3.jsonl 2>&1
$B --config C3 > $O/C3.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adjoint_kernel -c 2 -o $O/adjoint_C4 python bench.py --config C4 --path adjoint --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_adjoint.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:backsub_kernel -c 1 -o $O/backsub_C4 python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_backsub.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:sweep_kernel<\(int\)16' -c 1 -o $O/gt_C5 python bench.py --config C5 --slab 0/8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_gt.log 2>&1
ls -la $O
