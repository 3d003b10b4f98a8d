#!/bin/bash
# round-2 ncu evidence on the final code: the adjoint kernels on C4 (rhs over-read check) and the GT sweep on the
# C5 slab (DRAM traffic of the elements larger than one SM)
N=gpurun_out/ncu2; mkdir -p $N
#timeout 300 python bench.py --config C4 --path adjoint --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $N/plain_adjoint.log 2>&1 && \
#timeout 900 ncu --set full --clock-control none --import-source on -k regex:adjoint_kernel -c 2 -o $N/adjoint_C4 python bench.py --config C4 --path adjoint --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $N/ncu_adjoint.log 2>&1
timeout 300 python bench.py --config C5 --slab 0/8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $N/plain_c5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"sweep_kernel<16" -c 2 -o $N/gt_C5 python bench.py --config C5 --slab 0/8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $N/ncu_gt.log 2>&1
ls -la $N
