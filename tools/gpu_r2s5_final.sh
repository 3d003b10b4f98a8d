#!/bin/bash
# round 2, session 5: final evidence on the committed kernels. Order: GPU suite + smoke, the ncu --set full captures
# (summarised on the box so profiles/traffic.json matches the sources before the bench lines read it), every bench
# line, the C4 launch list. Everything lands in gpurun_out/s5f (profiles/ of the box copied there too).
O=gpurun_out/s5f; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
Q="--no-e2e --no-cpu-baseline"
timeout 300 python tools/prof_case.py --config C4 --reps 2 > $O/plain_prof_C4.log 2>&1 && {
timeout 900 $NCU -k regex:sweep_kernel -s 1 -c 1 -o $O/sweep_C4 -f python tools/prof_case.py --config C4 --reps 2 > $O/ncu_sweep.log 2>&1
timeout 600 $NCU -k regex:backsub_kernel -s 1 -c 1 -o $O/backsub_C4 -f python tools/prof_case.py --config C4 --reps 2 > $O/ncu_backsub.log 2>&1
}
timeout 300 python tools/prof_case.py --config C3 --reps 2 > $O/plain_prof_C3.log 2>&1 && \
timeout 900 $NCU -k regex:condense_kernel -s 1 -c 1 -o $O/panel_C3 -f python tools/prof_case.py --config C3 --reps 2 > $O/ncu_panel.log 2>&1
timeout 300 python tools/prof_case.py --config C2 --reps 2 > $O/plain_prof_C2.log 2>&1 && \
timeout 600 $NCU -k regex:warp_kernel -s 1 -c 1 -o $O/warp_C2 -f python tools/prof_case.py --config C2 --reps 2 > $O/ncu_warp.log 2>&1
timeout 300 python bench.py --config C4 --path adjoint --steps 1 --warmup 1 $Q > $O/plain_adjoint.log 2>&1 && \
timeout 900 $NCU -k regex:adjoint_kernel -c 2 -o $O/adjoint_C4 -f python bench.py --config C4 --path adjoint --steps 1 --warmup 1 $Q > $O/ncu_adjoint.log 2>&1
timeout 300 python bench.py --config C4 --path saved --steps 1 --warmup 1 $Q > $O/plain_saved.log 2>&1 && \
timeout 900 $NCU -k regex:"backsub_saved_kernel|save_kernel" -c 2 -o $O/saved_C4 -f python bench.py --config C4 --path saved --steps 1 --warmup 1 $Q > $O/ncu_saved.log 2>&1
timeout 300 python bench.py --config C5 --slab 0/8 --steps 1 --warmup 1 $Q > $O/plain_c5.log 2>&1 && \
timeout 1200 $NCU -k regex:"sweep_kernel<.int.16" -c 2 -o $O/gt_C5 -f python bench.py --config C5 --slab 0/8 --steps 1 --warmup 1 $Q > $O/ncu_gt.log 2>&1
R=""; add() { [ -f $O/$1.ncu-rep ] && R="$R --rep $O/$1.ncu-rep --config $2 --kernel $3"; }
add sweep_C4 C4 sweep_kernel; add backsub_C4 C4 backsub_kernel; add panel_C3 C3 condense_kernel; add warp_C2 C2 warp_kernel
add adjoint_C4 C4rhs "adjoint_kernel<0>"; add adjoint_C4 C4recon "adjoint_kernel<1>"
add saved_C4 C4 save_kernel; add saved_C4 C4 backsub_saved_kernel; add gt_C5 C5slab_ne252 "sweep_kernel<16"
python tools/summarize_profiles.py --tag r02 $R > $O/summarize.log 2>&1
python - >> $O/summarize.log 2>&1 <<'PY'
import json
p = "profiles/traffic.json"; t = json.load(open(p))
for old, new in (("C4rhs_adjoint", "C4_adjoint_rhs"), ("C4recon_adjoint", "C4_adjoint_recon")):
    if old in t: t[new] = t.pop(old)
json.dump(t, open(p, "w"), indent=1, sort_keys=True); print(sorted(t))
PY
bash tools/gpu_r2_evidence.sh > $O/evidence_summary.txt 2>&1
mkdir -p $O/r02; cp gpurun_out/r02/* $O/r02/ 2>/dev/null
timeout 300 python bench.py --steps 2 --warmup 3 $Q > $O/plain_default.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv python bench.py --steps 2 --warmup 3 $Q > $O/ncu_launches.log 2>&1
python tools/summarize_profiles.py --tag r02 --launches $O/launches_C4.csv --launch-config C4 >> $O/summarize.log 2>&1
mkdir -p $O/profiles; cp profiles/traffic.json profiles/r02_*_ncu.md profiles/r02_launches_C4.md $O/profiles/ 2>/dev/null
cp $O/launches_C4.csv $O/profiles/r02_launches_C4.csv 2>/dev/null
for f in $O/*.ncu-rep; do case $f in *sweep_C4*) ;; *) rm -f $f;; esac; done; du -sh $O; ls $O | head -60
