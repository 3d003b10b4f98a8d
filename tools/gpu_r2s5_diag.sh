#!/bin/bash
# round 2, session 5 diagnostics kept under profiles/r02: the per-bucket kernel times of the C5 slab and of the C4
# mesh at p = 4 (HDG_BUCKET_TIMES=1, synchronizing: never a bench value), and the clock64 cycle trace of one C4
# element in the sweep kernel (chain warp and one worker, per panel)
O=gpurun_out/s5d; mkdir -p $O
Q="--no-e2e --no-cpu-baseline"
HDG_BUCKET_TIMES=1 timeout 600 python bench.py --config C5 --slab 0/8 --steps 1 --warmup 1 $Q > $O/bucket_C5slab.out 2> $O/bucket_C5slab.err
grep HDG_BUCKET_TIMES $O/bucket_C5slab.err | tail -40 > $O/bucket_times_C5slab.txt
HDG_BUCKET_TIMES=1 timeout 600 python bench.py --config C4 --degree 4 --steps 1 --warmup 1 $Q > $O/bucket_C4p4.out 2> $O/bucket_C4p4.err
grep HDG_BUCKET_TIMES $O/bucket_C4p4.err | tail -4 > $O/bucket_times_C4p4.txt
timeout 300 python tools/trace_sweep.py --config C4 > $O/trace_sweep_C4.txt 2>&1
timeout 300 python tools/trace_condense.py --config C3 > $O/trace_panel_C3.txt 2>&1
tail -30 $O/trace_sweep_C4.txt; cat $O/bucket_times_C5slab.txt | tail -20
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 1200 $NCU -k regex:"sweep_kernel<.int.16" -c 2 -o $O/gt_C5 -f python bench.py --config C5 --slab 0/8 --steps 1 --warmup 1 $Q > $O/ncu_gt.log 2>&1
python tools/summarize_profiles.py --tag r02 --rep $O/gt_C5.ncu-rep --config C5slab_ne252 --kernel "sweep_kernel<16" > $O/summarize.log 2>&1
mkdir -p $O/profiles; cp profiles/traffic.json profiles/r02_condense_sweep_C5slab_ne252_ncu.md $O/profiles/; rm -f $O/gt_C5.ncu-rep
