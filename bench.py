#!/usr/bin/env python
"""bench.py — one step of the hybridization hot path per iteration, timed on the device.

A step (SURVEY.md §8(a) rows a1-a8 over one batch): hdg_condense (stage, LU with partial pivoting, local solves,
Schur complement, factor store) -> hdg_assemble_skeleton (+ shared-face exchange and accumulate when N > 1)
-> hdg_backsubstitute with a seeded trace vector lambda. The plan (row a0) is built once, outside the timed
region, as in a Newton loop on a fixed mesh.

Workload: BASELINE.json configs[3] ("C4", NS mixed HDG p=3, 131072 triangles, n_e=120, n_f=48) by default — the
largest configuration that fits one B200 (C5 needs ~490 GB). Synthetic inputs from the seeded generator, created
directly in HBM (bit-identical to the host generator the oracle uses). Inputs (~30 GB) exceed L2 (126 MB), so no
L2 flush is needed between steps; for workloads under 4x L2 (C1, C2) a 512 MB buffer is written before every
timed step and the steps are timed alone.

Contract: python bench.py --gpus N --steps K --warmup W [--impl reference] ; torchrun for N > 1 (one rank per
GPU, element slabs, NCCL for the shared-face exchange). Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "element condensations/s + back-subs/s (fp64), % of FP64/HBM roofline"


def algorithmic(ne, nf):
    """SURVEY.md §8(d) per-element work (one HBM pass; nothing the method avoids)."""
    ne = np.asarray(ne, dtype=np.float64)
    nf = np.asarray(nf, dtype=np.float64)
    cf = ne * (ne - 1) * (4 * ne + 1) / 6 + (nf + 1) * (2 * ne * ne - ne) + 2 * nf * ne * (nf + 1)
    cb = 8 * (ne * ne + 2 * ne * nf + nf * nf + ne + nf) + 8 * (nf * nf + nf) + (8 * ne * ne + 4 * ne)
    bf = 2 * ne * nf + 2 * ne * ne
    bb = 8 * (ne * ne + ne * nf + 2 * ne + nf) + 4 * ne
    return dict(condense_flops=float(cf.sum()), condense_bytes=float(cb.sum()), backsub_flops=float(bf.sum()),
                backsub_bytes=float(bb.sum()))


def run_adjoint(args, wl, rank, world, local):
    """The adjoint (transposed) step on the primal factors — g~ = r~_f - B^T A^-T r~_e, K~ = sum S_e^T, E~ = sum g~,
    u~ = A^-T (r~_e - C^T lambda~) — timed like the primal step (with N > 1 the S_e^T strips of
    shared faces travel through the same transport as the primal's)."""
    import torch
    import torch.distributed as dist
    import paper_1308_3995_b200 as hdg
    w, ctx, stream, inp, lam = wl["w"], wl["ctx"], wl["stream"], wl["inp"], wl["lam"]
    S, F, infot, K, E = (wl[k] for k in ("S", "F", "infot", "K", "E"))
    eb, n = wl["eb"], wl["n"]
    gt, ut = ctx.alloc("g"), ctx.alloc("u")
    ctx.condense(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], S, wl["g"], F, infot, stream=stream)
    rt, lam_t = inp["re"], lam      # seeded stand-ins for the functional's linearization and the adjoint trace
    launches = [0]

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        ctx.condense_adjoint_rhs(F, inp["B"], rt, None, gt, stream=stream)
        launches[0] += ctx.launch_count()
        if ev:
            ev[1].record(stream)
        ctx.assemble_adjoint(S, gt, K, E, send=wl["send"], stream=stream)
        launches[0] += ctx.launch_count()
        if wl["exchange"] and not ctx.has_comm:   # (with its own communicator the library exchanged already)
            hdg.exchange(ctx, wl["send"], wl["recv"], stream=stream)
            ctx.skeleton_accumulate(wl["recv"], K, E, stream=stream)
            launches[0] += ctx.launch_count()
        if ev:
            ev[2].record(stream)
        ctx.backsubstitute_adjoint(F, inp["C"], rt, lam_t, ut, stream=stream)
        launches[0] += ctx.launch_count()
        if ev:
            ev[3].record(stream)

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    launches[0] = 0
    for i in range(args.steps):
        step(evs[i])
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    t = torch.tensor([sum(e[0].elapsed_time(e[1]) for e in evs), sum(e[1].elapsed_time(e[2]) for e in evs),
                      sum(e[2].elapsed_time(e[3]) for e in evs), sum(e[0].elapsed_time(e[3]) for e in evs)],
                     dtype=torch.float64, device=torch.device("cuda", local)) / args.steps
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    rhs_ms, asm_ms, bs_ms, ms_step = t.tolist()
    ne = np.asarray(w.elem_ne[eb:eb + n], dtype=np.float64)
    nf = np.asarray(w.elem_nf[eb:eb + n], dtype=np.float64)
    fac = 8 * ne * ne + 4 * ne
    rhs_bytes = float((fac + 8 * ne * nf + 8 * ne + 8 * nf).sum())        # factors, B, r~_e, g~
    bs_bytes = float((fac + 8 * nf * ne + 16 * ne + 8 * nf).sum())        # factors, C, r~_e, lambda~_e, u~
    hbm = measured_peaks().get("hbm_gbs") or 6551.4
    ach = (rhs_bytes + bs_bytes) / ((rhs_ms + bs_ms) * 1e-3) / 1e9
    elems = n if args.slab is not None else w.E
    line = {"metric": "adjoint element steps/s (fp64): adjoint rhs + K^T assembly + adjoint reconstruction",
            "value": elems / (ms_step * 1e-3), "unit": "elements/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "impl": "hdg", "path": "adjoint",
            "data": "synthetic (seeded Philox blocks; r~_e, lambda~ seeded stand-ins)",
            "config": {"workload": args.config + (f" mesh at p = {args.degree}" if args.degree else ""),
                       "elements": int(n), "n_e": int(ne.max()), "n_f": int(nf.max()),
                       "step": "condense_adjoint_rhs + assemble_adjoint + backsubstitute_adjoint"},
            "adjoint_rhs_ms": rhs_ms, "assemble_adjoint_ms": asm_ms, "backsub_adjoint_ms": bs_ms,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                         "traffic": _traffic(args.config + "_adjoint_rhs") if args.degree is None else None,
                         "traffic_kernel": "adjoint_kernel<0> (dram read + write per launch, ncu --set full)",
                         "kernel": "adjoint_kernel<0, 1> (adjoint.cu)",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                         "bytes_per_step": rhs_bytes + bs_bytes},
            "gpu_launches": launches[0], "clocks": clk, "e2e": None, "cpu_baseline": None}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def run_solve(args, wl, rank, world, local):
    """The Newton step with the skeleton solve in it (§8(f) NEXT #3): condense -> assemble -> solve K lambda = E
    (block-Jacobi GMRES, rtol 1e-10, from lambda = 0) -> back-substitute with the computed lambda. Reports the solve
    time, its iterations and the SpMV's HBM rate (K's values + column gathers per iteration)."""
    import torch
    import torch.distributed as dist
    w, ctx, stream, inp = wl["w"], wl["ctx"], wl["stream"], wl["inp"]
    info = wl["info"]
    lam = torch.zeros(w.n_trace, dtype=torch.float64, device=torch.device("cuda", local))
    y = ctx.alloc("E")
    res = []

    def step(timed):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(stream)
        ctx.condense(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], wl["S"], wl["g"], wl["F"],
                     wl["infot"], stream=stream)
        ev[1].record(stream)
        ctx.assemble_skeleton(wl["S"], wl["g"], wl["K"], wl["E"], stream=stream)
        ev[2].record(stream)
        lam.zero_()
        it, rr = ctx.skeleton_solve(wl["K"], wl["E"], lam, rtol=1e-10, maxit=2000, restart=40, stream=stream)
        ev[3].record(stream)
        ctx.backsubstitute(wl["F"], inp["B"], inp["re"], lam, wl["u"], stream=stream)
        ev[4].record(stream)
        torch.cuda.synchronize()
        if timed:
            res.append(([ev[i].elapsed_time(ev[i + 1]) for i in range(4)], it, rr))

    clocks = ClockSampler(local)
    clocks.start()                       # before the warm-up: nvidia-smi needs 0.1-0.3 s for its first sample
    for _ in range(args.warmup):
        step(False)
    clocks.mark()
    for _ in range(args.steps):
        step(True)
    clk = clocks.stop(replay=lambda: step(False))
    # one SpMV alone (HBM rate of the solver's dominant kernel)
    a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x = torch.randn(w.n_trace, dtype=torch.float64, device=lam.device)
    ctx.skeleton_spmv(wl["K"], x, y, stream=stream)
    a_.record(stream)
    for _ in range(10):
        ctx.skeleton_spmv(wl["K"], x, y, stream=stream)
    b_.record(stream)
    torch.cuda.synchronize()
    spmv_ms = a_.elapsed_time(b_) / 10
    spmv_bytes = 8.0 * info.nvals + 4.0 * info.nnzb + 8.0 * (info.nnzb + 1) + 16.0 * w.n_trace
    t = np.array([r[0] for r in res]).mean(axis=0)
    if world > 1:      # max over ranks
        tt = torch.tensor(t, dtype=torch.float64, device=lam.device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = tt.cpu().numpy()
    its = [r[1] for r in res]
    hbm = measured_peaks().get("hbm_gbs") or 6551.4
    line = {"metric": "Newton step with the skeleton solve (fp64): condense + assemble + GMRES + back-substitute",
            "value": w.E / (t.sum() * 1e-3), "unit": "elements/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(t.sum()), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "impl": "hdg", "path": "solve",
            "data": "synthetic (seeded Philox blocks with BASELINE.json distributions, generated in HBM)",
            "config": {"workload": args.config, "elements": w.E, "trace_dofs": w.n_trace, "nnz_blocks": info.nnzb,
                       "solver": "GMRES(40), right block-Jacobi, rtol 1e-10, lambda0 = 0" +
                                 (f"; distributed over {world} slabs (NCCL halo + all-reduce)" if world > 1 else "")},
            "condense_ms": float(t[0]), "assemble_ms": float(t[1]), "solve_ms": float(t[2]), "backsub_ms": float(t[3]),
            "solve_iterations": its, "solve_true_relres": [r[2] for r in res],
            "solve_ms_per_iteration": float(t[2]) / max(1, np.mean(its)),
            "spmv_ms": spmv_ms, "spmv_hbm_gbs": spmv_bytes / (spmv_ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": "spmv_kernel (skeleton_solve.cu)",
                         "achieved": spmv_bytes / (spmv_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": spmv_bytes / (spmv_ms * 1e-3) / 1e9 / hbm, "traffic": None,
                         "bytes_per_launch": spmv_bytes},
            "clocks": clk, "e2e": None, "cpu_baseline": None}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def _traffic(key):
    """DRAM read + write bytes per launch of the dominant kernel from the committed `ncu --set full` capture
    (profiles/traffic.json), only while the kernel's source is unchanged since that capture (same hash as
    tools/summarize_profiles.py recorded); otherwise None — a stale figure is never reported."""
    try:
        e = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(key)
    except Exception:
        return None
    if not isinstance(e, dict):
        return None
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    try:
        from summarize_profiles import source_sha
        return e["bytes"] if source_sha(e.get("kernel", "")) == e.get("source_sha") else None
    except Exception:
        return None


def measured_peaks():
    peaks = {}
    try:
        peaks.update(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))))
    except Exception:
        pass
    return peaks


def fp64_peak_in_run():
    """K9: FP64 peak measured on this box in this run (tools/peaks: DMMA and DFMA loops)."""
    exe = os.path.join(ROOT, "tools", "peaks")
    try:
        out = subprocess.run([exe, "fp64"], capture_output=True, text=True, timeout=120).stdout
        d = json.loads(out.strip().splitlines()[-1])
        dmma = max(v for k, v in d.items() if k.startswith("dmma"))
        dfma = max(v for k, v in d.items() if k.startswith("dfma"))
        return dmma, dfma
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"hdg_clocks_{os.getpid()}.csv")

    def start(self):
        """Started before the warm-up (nvidia-smi needs ~0.1-0.3 s to produce its first sample); mark() / stop()
        bracket the timed region and only samples inside it are kept (all of them if the region was too short)."""
        self.t_mark = None
        q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def mark(self):
        self.t_mark = time.time()

    def stop(self, replay=None):
        """replay: a callable re-running the timed step; for regions shorter than nvidia-smi's sampling (C1, C2)
        it is re-run for ~0.4 s after the timed region while the sampler keeps going, and the clocks are taken
        from that window (noted in the record)."""
        t_end = time.time()
        if self.proc is None:
            return None
        if replay is not None and t_end - (self.t_mark or t_end) < 0.3:
            t0 = time.time()
            while time.time() - t0 < 0.4:
                replay()
            self.t_mark, t_end = t0, time.time()
            self.replayed = True
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 10:
                try:
                    ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    rows.append((ts, float(f[2]), float(f[3]), f[6:10]))
                except ValueError:
                    pass
        if not rows:
            return {"samples": 0, "note": "no nvidia-smi sample"}
        inside = [r for r in rows if self.t_mark is not None and self.t_mark - 0.05 <= r[0] <= t_end + 0.05]
        note = None
        if getattr(self, "replayed", False):
            note = ("timed region shorter than the 100 ms sampling interval: clocks sampled while the same step "
                    "re-ran for 0.4 s right after it")
        if not inside:
            inside = rows[-3:]
            note = "timed region shorter than the 100 ms sampling interval: last samples of the warm-up and region"
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, _, r in inside for i in range(4) if r[i].lower() == "active"})
        out = {"sm_mhz": float(np.median([r[1] for r in inside])), "sm_max_mhz": max(r[2] for r in inside),
               "samples": len(inside), "reasons": reasons}
        if note:
            out["note"] = note
        return out


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def slab_bounds(E: int, n: int):
    return np.array([(r * E) // n for r in range(n + 1)], dtype=np.int64)


def _omp_threads(n=None):
    """OpenMP thread count of this process (the oracle's parallel loops): set it when n is given, return the
    previous value. Plumbing for the 1-thread oracle number; the oracle is not modified."""
    import ctypes
    try:
        gomp = ctypes.CDLL("libgomp.so.1")
    except OSError:
        return None
    prev = gomp.omp_get_max_threads()
    if n is not None:
        gomp.omp_set_num_threads(int(n))
    return prev


def oracle_sample(w, seconds: float, lam, max_elems=None, threads=None):
    """The oracle (as it stands) on a bounded sample of the workload: condense + assemble (rows owned by the
    sample) + back-substitute for the first m elements. Returns (elements/s, m, wall seconds, threads).
    threads: OpenMP threads for this sample (None: all the host cores, the default)."""
    import oracle
    import gen
    if threads is not None:
        prev = _omp_threads(threads)
        try:
            v = oracle_sample(w, seconds, lam, max_elems)
        finally:
            if prev:
                _omp_threads(prev)
        return v[0], v[1], v[2], threads

    def run(m):
        blk = gen.host_blocks(w, 0, m)
        t0 = time.perf_counter()
        c = oracle.condense(w.elem_ne[:m], w.elem_nf[:m], blk)
        f1 = int(np.searchsorted(w.face_elem[:, 0], m))      # faces whose left element is in the sample
        sym = oracle.symbolic(w.elem_face, w.face_elem, w.face_ndof, 0, f1)
        oracle.assemble(w.elem_face, w.face_ndof, w.face_off, w.elem_nf[:m], c["S"], c["off_S"], c["g"],
                        c["off_g"], sym, 0, f1, 0, m)
        oracle.backsub(w.elem_face, w.face_ndof, w.face_off, w.elem_ne[:m], w.elem_nf[:m], c["LU"], c["off_LU"],
                       c["piv"], c["off_piv"], blk["B"], blk["off_B"], blk["re"], blk["off_re"], lam)
        return time.perf_counter() - t0

    m = min(64, w.E)
    t = run(m)
    m2 = int(min(w.E, max(m, m * seconds / max(t, 1e-6))))
    if max_elems:
        m2 = min(m2, max_elems)
    t2 = run(m2)
    threads = _omp_threads() or int(os.environ.get("OMP_NUM_THREADS", len(os.sched_getaffinity(0))))
    return m2 / t2, m2, t2, threads


def run_reference(args, rank, world):
    """--impl reference: the oracle (the only reference this tier has) on the box's host cores."""
    if rank != 0:
        return
    import gen
    w = gen.config(args.config)
    lam = gen.host_lambda(w)
    for _ in range(args.warmup):
        oracle_sample(w, args.ref_seconds / 4, lam, max_elems=4096)
    vals, ms, secs = [], [], []
    for _ in range(args.steps):
        v, m, t, threads = oracle_sample(w, args.ref_seconds, lam)
        vals.append(v)
        ms.append(m)
        secs.append(t)
    value = float(np.median(vals))
    sample = (f"first {ms[-1]} of {w.E} elements of {args.config} per step: oracle condense + assemble (rows owned "
              f"by the sample) + back-substitute, {np.mean(secs):.1f} s per step, generation excluded")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * w.E / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Philox blocks, BASELINE.json distributions)",
            "config": {"workload": args.config, "elements": w.E, "n_e": int(w.elem_ne.max()),
                       "n_f": int(w.elem_nf.max())},
            "cpu_baseline": {"value": value, "unit": "elements/s", "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_of(config: str, degree=None):
    """The BASELINE config, or its mesh at another uniform polynomial degree (--degree: e.g. the adjoint's
    enriched degree p + 1)."""
    import gen
    if degree is None:
        return gen.config(config)
    c = gen.CONFIGS[config]
    return gen.make_workload(f"{config}-p{degree}", nr=c["nr"], nt=c["nt"], m_elem=c["m_elem"], p_fixed=int(degree),
                             seed=gen.SEED_BASE + 1 + list(gen.CONFIGS).index(config))


def setup_workload(config: str, rank: int = 0, world: int = 1, local: int = 0, slab=None, degree=None):
    """The benchmark's launch configuration (shared with the full-size parity tests): this rank's element slab of
    the BASELINE config, inputs generated directly in HBM (bit-identical to gen.host_blocks), plan built once,
    outputs allocated. slab = (r, P): emulate rank r of a P-way partition on this single GPU (used for C5, whose
    full mesh needs ~490 GB: rank 0 of 8 is one B200's share at N = 8; its shared-face rows get only the local
    contributions, the exchange step is not run)."""
    import torch
    import gen
    import paper_1308_3995_b200 as hdg
    dev = torch.device("cuda", local)
    w = workload_of(config, degree)
    if slab is not None:
        r_emul, p_emul = slab
        reb = slab_bounds(w.E, p_emul)
        eb, n = int(reb[r_emul]), int(reb[r_emul + 1] - reb[r_emul])
        ctx = hdg.Context(local, r_emul, p_emul)
        info = ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne, eb, n, reb)
    else:
        reb = slab_bounds(w.E, world)
        eb, n = int(reb[rank]), int(reb[rank + 1] - reb[rank])
        # N > 1: the context owns an NCCL communicator; hdg_assemble_skeleton packs, exchanges (grouped
        # ncclSend/ncclRecv on the step's stream) and accumulates the shared-face rows itself
        ctx = hdg.nccl_context(local, rank, world) if world > 1 else hdg.Context(local, rank, world)
        info = ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne, eb, n, reb if world > 1 else None)
    stream = torch.cuda.Stream(dev)
    inp = {}
    with torch.cuda.stream(stream):
        dne = torch.from_numpy(w.elem_ne[eb:eb + n].copy()).to(dev)
        dnf = torch.from_numpy(w.elem_nf[eb:eb + n].copy()).to(dev)
        for k in ("A", "B", "C", "D", "re", "rf"):
            o = w.off[k][eb:eb + n + 1] - w.off[k][eb]
            inp[k] = torch.empty(max(int(o[-1]), 2), dtype=torch.float64, device=dev)
            if w.uniform:
                gen.device_blocks(w, k, inp[k], e0=eb, n=n, stream=stream.cuda_stream)
            else:
                gen.device_blocks(w, k, inp[k], e0=eb, n=n, off=torch.from_numpy(o).to(dev), stream=stream.cuda_stream,
                                  dev_ne=dne, dev_nf=dnf)
        lam = torch.empty(w.n_trace, dtype=torch.float64, device=dev)
        gen.device_lambda(w, lam, torch.from_numpy(w.face_ndof).to(dev), torch.from_numpy(w.face_off).to(dev))
    out = dict(w=w, ctx=ctx, info=info, stream=stream, inp=inp, lam=lam, eb=eb, n=n, reb=reb, world=world,
               exchange=(world > 1 and slab is None))
    for k in ("S", "g", "u", "factors", "info", "K", "E"):
        out[{"factors": "F", "info": "infot"}.get(k, k)] = ctx.alloc(k)
    own = ctx.has_comm
    out["send"] = ctx.alloc("send") if info.send_doubles > 0 and not own else None
    out["recv"] = ctx.alloc("recv") if info.recv_doubles > 0 and not own else None
    return out


def run_chunked(args, rank, world, local, dmma_peak):
    """C5 (configs[4], ~490 GB) on N GPUs, whole mesh: the mesh is cut into V = max(8, N) element slabs ("virtual
    ranks"); rank r processes its V/N slabs one after another, each slab's inputs generated in HBM
    (outside the timed region: "C5 at P = 1, 2: sum of per-chunk kernel times; generation and H2D
    excluded"), condensed, assembled (its K rows stay resident) and back-substituted. The shared-face exchange
    between slabs follows once per step: slabs on the same GPU by device copies, slabs on other GPUs through
    torch.distributed point-to-point (NCCL); then every slab's ordered accumulate. Step time = the sum of the
    slabs' condense + assemble + back-substitute times + the exchange/accumulate time, max over ranks."""
    import torch
    import torch.distributed as dist
    import gen
    import paper_1308_3995_b200 as hdg
    dev = torch.device("cuda", local)
    w = gen.config(args.config)
    V = max(8, world)
    if V % world:
        raise SystemExit(f"--gpus {world}: the {V} C5 slabs must divide evenly over the ranks")
    vb = slab_bounds(w.E, V)
    mine = list(range(rank * V // world, (rank + 1) * V // world))
    owner = lambda v: v * world // V                                     # noqa: E731
    stream = torch.cuda.Stream(dev)
    sl = {}
    for v in mine:
        eb, n = int(vb[v]), int(vb[v + 1] - vb[v])
        ctx = hdg.Context(local, v, V)
        info = ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne, eb, n, vb)
        sl[v] = dict(ctx=ctx, info=info, eb=eb, n=n, K=ctx.alloc("K"), E=ctx.alloc("E"), send=ctx.alloc("send"),
                     recv=ctx.alloc("recv"), counts=ctx.exchange_counts())
    # per-slab work buffers, sized for the largest owned slab, reused slab after slab
    keys = ("A", "B", "C", "D", "re", "rf")
    big = {k: max(int(w.off[k][sl[v]["eb"] + sl[v]["n"]] - w.off[k][sl[v]["eb"]]) for v in mine) for k in keys}
    inp = {k: torch.empty(max(big[k], 2), dtype=torch.float64, device=dev) for k in keys}
    outs = {k: max(getattr(sl[v]["info"], f) for v in mine) for k, f in (("S", "len_S"), ("g", "len_g"),
                                                                          ("u", "len_u"), ("F", "factor_bytes"))}
    S = torch.empty(outs["S"], dtype=torch.float64, device=dev)
    g = torch.empty(outs["g"], dtype=torch.float64, device=dev)
    u = torch.empty(outs["u"], dtype=torch.float64, device=dev)
    F = torch.empty(outs["F"], dtype=torch.uint8, device=dev)
    infot = torch.empty(max(sl[v]["n"] for v in mine), dtype=torch.int32, device=dev)
    lam = torch.empty(w.n_trace, dtype=torch.float64, device=dev)
    with torch.cuda.stream(stream):
        gen.device_lambda(w, lam, torch.from_numpy(w.face_ndof).to(dev), torch.from_numpy(w.face_off).to(dev))
    dne = {v: torch.from_numpy(w.elem_ne[sl[v]["eb"]:sl[v]["eb"] + sl[v]["n"]].copy()).to(dev) for v in mine}
    dnf = {v: torch.from_numpy(w.elem_nf[sl[v]["eb"]:sl[v]["eb"] + sl[v]["n"]].copy()).to(dev) for v in mine}
    doff = {(v, k): torch.from_numpy(w.off[k][sl[v]["eb"]:sl[v]["eb"] + sl[v]["n"] + 1] - w.off[k][sl[v]["eb"]]).to(dev)
            for v in mine for k in keys}
    torch.cuda.synchronize()
    launches = [0]

    def step(timed):
        evs = []
        for v in mine:
            x = sl[v]
            with torch.cuda.stream(stream):      # generation of this slab's inputs: outside the timed region
                for k in keys:
                    gen.device_blocks(w, k, inp[k], e0=x["eb"], n=x["n"], off=doff[(v, k)], stream=stream.cuda_stream,
                                      dev_ne=dne[v], dev_nf=dnf[v])
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ctx = x["ctx"]
            e[0].record(stream)
            ctx.condense(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], S, g, F, infot, stream=stream)
            launches[0] += ctx.launch_count()
            e[1].record(stream)
            ctx.assemble_skeleton(S, g, x["K"], x["E"], send=x["send"], stream=stream)
            launches[0] += ctx.launch_count()
            e[2].record(stream)
            ctx.backsubstitute(F, inp["B"], inp["re"], lam, u, stream=stream)
            launches[0] += ctx.launch_count()
            e[3].record(stream)
            evs.append(e)
        # a7 between slabs: same-GPU peers by copies, other GPUs by NCCL point-to-point (one canonical order of
        # (source slab, destination slab) pairs on every rank, so the messages between two ranks match)
        ex = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ex[0].record(stream)
        with torch.cuda.stream(stream):
            ops = []
            for src in range(V):
                for dst in range(V):
                    if src == dst:
                        continue
                    so, do = owner(src), owner(dst)
                    if so != rank and do != rank:
                        continue
                    if so == rank:
                        sc, sd, _, _ = sl[src]["counts"]
                        cnt, off = int(sc[dst]), int(sd[dst])
                    else:
                        _, _, rc, rd = sl[dst]["counts"]
                        cnt, off = int(rc[src]), int(rd[src])
                    if cnt == 0:
                        continue
                    if so == rank and do == rank:
                        _, _, rc, rd = sl[dst]["counts"]
                        sl[dst]["recv"][int(rd[src]):int(rd[src]) + cnt].copy_(sl[src]["send"][off:off + cnt])
                    elif so == rank:
                        ops.append(dist.P2POp(dist.isend, sl[src]["send"][off:off + cnt], do))
                    else:
                        ops.append(dist.P2POp(dist.irecv, sl[dst]["recv"][off:off + cnt], so))
            if ops:
                for wk in dist.batch_isend_irecv(ops):
                    wk.wait()
            for v in mine:
                sl[v]["ctx"].skeleton_accumulate(sl[v]["recv"], sl[v]["K"], sl[v]["E"], stream=stream)
                launches[0] += sl[v]["ctx"].launch_count()
        ex[1].record(stream)
        torch.cuda.synchronize()
        if not timed:
            return None
        cond = sum(e[0].elapsed_time(e[1]) for e in evs)
        asm = sum(e[1].elapsed_time(e[2]) for e in evs)
        bs = sum(e[2].elapsed_time(e[3]) for e in evs)
        xch = ex[0].elapsed_time(ex[1])
        return cond, asm, bs, xch

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step(False)
    for v in mine:
        bad, code = sl[v]["ctx"].first_error(infot[:sl[v]["n"]], stream=stream)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    launches[0] = 0
    res = [step(True) for _ in range(args.steps)]
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    t = torch.tensor([sum(r[i] for r in res) / args.steps for i in range(4)], dtype=torch.float64, device=dev)
    t_step = torch.tensor([sum(res[-1])], dtype=torch.float64, device=dev)
    tot = torch.tensor([sum(sum(r) for r in res) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    cond_ms, asm_ms, bs_ms, x_ms = t.tolist()
    ms_step = tot.item()
    if rank == 0:
        ne = w.elem_ne[int(vb[mine[0]]):int(vb[mine[-1] + 1])]
        nf = w.elem_nf[int(vb[mine[0]]):int(vb[mine[-1] + 1])]
        work = algorithmic(ne, nf)
        fp64_peak = dmma_peak or 37.2
        ach = work["condense_flops"] / (cond_ms * 1e-3) / 1e12
        line = {"metric": METRIC, "value": w.E / (ms_step * 1e-3), "unit": "elements/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded Philox blocks with BASELINE.json distributions, generated in HBM per slab)",
                "config": {"workload": f"C5 whole mesh ({w.E} elements) in {V} slabs, {len(mine)} per GPU",
                           "elements": w.E, "n_e": int(w.elem_ne.max()), "n_f": int(w.elem_nf.max()),
                           "parallelism": f"element slabs x{world} (x{len(mine)} chunks per GPU)",
                           "l2": "inputs exceed the 126 MB L2; no flush needed",
                           "step": "per slab: condense + assemble_skeleton + backsubstitute; then the shared-face "
                                   "exchange between slabs + ordered accumulate",
                           "timing": "sum of the per-slab CUDA-event times + exchange; slab input generation "
                                     "excluded (SURVEY.md §8(d))"},
                "condense_ms": cond_ms, "assemble_ms": asm_ms, "backsub_ms": bs_ms, "exchange_ms": x_ms,
                "condense_per_s": w.E / (cond_ms * 1e-3 * world / world), "backsub_per_s": w.E / (bs_ms * 1e-3),
                "roofline": {"bound": "tensor", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                             "frac": ach / fp64_peak, "traffic": None,
                             "kernel": "hdg_condense over C5's hp buckets (sweep GT / sweep / panel / warp)",
                             "flops_per_rank_step": work["condense_flops"]},
                "gpu_launches": launches[0] // max(1, args.steps) * args.steps, "clocks": clk,
                "cpu_baseline": None, "e2e": None}
        print(json.dumps(line), flush=True)
    return 0



def run_step(wl, ev=None):
    """One step of the hot path on the workload; returns the libhdg launches issued."""
    import paper_1308_3995_b200 as hdg
    ctx, stream, inp = wl["ctx"], wl["stream"], wl["inp"]
    n = 0
    if ev:
        ev[0].record(stream)
    if wl.get("fused"):
        # §8(f) NEXT #2: condensation and assembly fused (S_e, g_e straight into K, E; bitwise the same K, E)
        ctx.condense_assemble(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], wl["K"], wl["E"], wl["F"],
                              wl["infot"], stream=stream)
        n += ctx.launch_count()
        if ev:
            ev[1].record(stream)
            ev[2].record(stream)
        ctx.backsubstitute(wl["F"], inp["B"], inp["re"], wl["lam"], wl["u"], stream=stream)
        n += ctx.launch_count()
        if ev:
            ev[3].record(stream)
        return n
    if wl.get("X") is not None:
        # §8(f) NEXT #2: the condensation also saves X = A^-1 [B | r_e] (written by the kernels that
        # form it; a save pass on the fresh factors for the others)
        ctx.condense_saved(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], wl["S"], wl["g"], wl["F"],
                           wl["X"], wl["infot"], stream=stream)
    else:
        ctx.condense(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], wl["S"], wl["g"], wl["F"],
                     wl["infot"], stream=stream)
    n += ctx.launch_count()
    if ev:
        ev[1].record(stream)
    ctx.assemble_skeleton(wl["S"], wl["g"], wl["K"], wl["E"], send=wl["send"], stream=stream)
    n += ctx.launch_count()
    if wl["exchange"] and not ctx.has_comm:   # (with its own communicator the library exchanged already)
        hdg.exchange(ctx, wl["send"], wl["recv"], stream=stream)
        ctx.skeleton_accumulate(wl["recv"], wl["K"], wl["E"], stream=stream)
        n += ctx.launch_count()
    if ev:
        ev[2].record(stream)
    if wl.get("X") is not None:
        # §8(f) NEXT #2: the local solutions were saved after the condensation (ev[4]..ev[5]);
        # the reconstruction is a GEMV on them
        ctx.backsubstitute_saved(wl["X"], wl["lam"], wl["u"], stream=stream)
    else:
        ctx.backsubstitute(wl["F"], inp["B"], inp["re"], wl["lam"], wl["u"], stream=stream)
    n += ctx.launch_count()
    if ev:
        ev[3].record(stream)
    return n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hdg", choices=["hdg", "reference"])
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--path", default="primal", choices=["primal", "adjoint", "saved", "solve", "fused"],
                    help="adjoint: time the transposed path (SURVEY.md §8(f) NEXT #1) on the primal factors; saved: "
                         "save the local solutions after the condensation and reconstruct from them (NEXT #2)")
    ap.add_argument("--degree", type=int, default=None,
                    help="run the config's mesh at this uniform degree (C1-C4; e.g. the adjoint at p + 1)")
    ap.add_argument("--graph", type=int, default=0,
                    help="also time G back-to-back steps captured in one CUDA graph (launch latency; C1/C2)")
    ap.add_argument("--slab", default=None,
                    help="r/P: time rank r's slab of a P-way partition on this one GPU (default for C5: 0/8)")
    args = ap.parse_args()
    if args.slab is not None:
        r_, p_ = (int(x) for x in args.slab.split("/"))
        args.slab = (r_, p_)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import gen
    import paper_1308_3995_b200 as hdg

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    dmma_peak, dfma_peak = (fp64_peak_in_run() if rank == 0 else (None, None))

    if args.config == "C5" and args.slab is None:
        # C5 (~490 GB of inputs) does not fit one B200: the whole mesh in element slabs, several per GPU
        return run_chunked(args, rank, world, local, dmma_peak)
    wl = setup_workload(args.config, rank, world, local, slab=args.slab, degree=args.degree)
    if args.path == "adjoint":
        return run_adjoint(args, wl, rank, world, local)
    if args.path == "solve":
        return run_solve(args, wl, rank, world, local)
    if args.path == "saved":
        wl["X"] = wl["ctx"].alloc("X")
    if args.path == "fused":
        if world > 1:
            raise SystemExit("--path fused: single rank (hdg_condense_assemble)")
        wl["fused"] = True
    w, ctx, info, stream, inp, lam = wl["w"], wl["ctx"], wl["info"], wl["stream"], wl["inp"], wl["lam"]
    S, g, u, F, infot, K, E, send, recv = (wl[k] for k in ("S", "g", "u", "F", "infot", "K", "E", "send", "recv"))
    eb, n, reb = wl["eb"], wl["n"], wl["reb"]
    elems = n if args.slab is not None else w.E     # elements one step processes (all ranks together)
    workload = args.config if args.slab is None else (f"{args.config} slab {args.slab[0]}/{args.slab[1]} "
                                                      f"(elements [{eb}, {eb + n}) of {w.E})")
    torch.cuda.synchronize()

    launches = [0]
    # inputs smaller than L2 (C1): flush L2 before every timed step by writing a 512 MB buffer on the same
    # stream, and time the steps alone (per-step events) so the flush stays outside the measurement
    in_bytes = sum(v.numel() for v in inp.values()) * 8
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev) if in_bytes < 4 * 126e6 else None

    def step(ev=None):
        if flush is not None and ev is not None:
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
        launches[0] += run_step(wl, ev)

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    bad, code = ctx.first_error(infot, stream=stream)
    if bad >= 0:
        raise RuntimeError(f"singular element {bad} (info {code}) in the benchmark inputs")

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    launches[0] = 0
    t0.record(stream)
    for i in range(args.steps):
        step(evs[i])
    t1.record(stream)
    torch.cuda.synchronize()

    def _replay():
        step()
        torch.cuda.synchronize()

    clk = clocks.stop(replay=_replay)
    if world > 1:
        dist.barrier()
    total_ms = t0.elapsed_time(t1) if flush is None else sum(e[0].elapsed_time(e[3]) for e in evs)
    cond_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    asm_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    bs_ms = sum(e[2].elapsed_time(e[3]) for e in evs) / args.steps
    gpu_launches = launches[0]
    t = torch.tensor([total_ms, cond_ms, asm_ms, bs_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, cond_ms, asm_ms, bs_ms = t.tolist()
    ms_step = total_ms / args.steps

    # ---- CUDA graph of G back-to-back steps (no flush between them): separates launch latency
    graph = None
    if args.graph > 0:
        g_ = torch.cuda.CUDAGraph()
        run_step(wl)                      # warm (kernel attributes set outside the capture)
        torch.cuda.synchronize()
        with torch.cuda.graph(g_, stream=stream):
            for _ in range(args.graph):
                run_step(wl)
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):     # replay() launches on the current stream: make it the timed one
            g_.replay()
            torch.cuda.synchronize()
            a_.record(stream)
            g_.replay()
            b_.record(stream)
        torch.cuda.synchronize()
        gms = a_.elapsed_time(b_) / args.graph
        graph = {"steps_in_graph": args.graph, "ms_per_step": gms, "value": elems / (gms * 1e-3),
                 "unit": "elements/s", "note": "back to back inside one CUDA graph, L2 not flushed between steps"}

    # ---- e2e: the same step through the public API with HOST buffers (pinned), copies inside the timed region ----
    e2e = None
    if not args.no_e2e:
        host = {k: torch.empty(v.numel(), dtype=v.dtype, pin_memory=True) for k, v in inp.items()}
        for k in host:
            host[k].copy_(inp[k])
        hlam = torch.empty(lam.numel(), dtype=torch.float64, pin_memory=True)
        hlam.copy_(lam)
        hu = torch.empty(u.numel(), dtype=torch.float64, pin_memory=True)
        hK = torch.empty(K.numel(), dtype=torch.float64, pin_memory=True)
        hE = torch.empty(E.numel(), dtype=torch.float64, pin_memory=True)
        h2d = sum(v.numel() * 8 for v in host.values()) + hlam.numel() * 8
        d2h = (hu.numel() + hK.numel() + hE.numel()) * 8

        def e2e_step():
            with torch.cuda.stream(stream):
                for k in host:
                    inp[k].copy_(host[k], non_blocking=True)
                lam.copy_(hlam, non_blocking=True)
            step()
            with torch.cuda.stream(stream):
                hK.copy_(K, non_blocking=True)
                hE.copy_(E, non_blocking=True)
                hu.copy_(u, non_blocking=True)

        ke2e = max(1, min(args.steps, 3))
        e2e_step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        a.record(stream)
        for _ in range(ke2e):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([a.elapsed_time(b) / ke2e], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": elems / (te.item() / 1e3), "unit": "elements/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": ke2e,
               "note": "host (pinned) inputs A,B,C,D,r_e,r_f,lambda copied in and K,E,u copied out every step"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, m, secs, threads = oracle_sample(w, args.cpu_seconds, gen.host_lambda(w))
        v1, m1, secs1, _ = oracle_sample(w, 3.0, gen.host_lambda(w), threads=1)
        cpu = {"value": v, "unit": "elements/s", "cores": threads, "kind": "oracle",
               "sample": f"first {m} of {w.E} elements: oracle condense + assemble (rows owned by the sample) + "
                         f"back-substitute, {secs:.1f} s wall, generation excluded",
               "one_thread": {"value": v1, "unit": "elements/s", "cores": 1,
                              "sample": f"first {m1} elements, {secs1:.1f} s wall, 1 OpenMP thread"},
               "host_cpu": _cpu_model()}

    if rank == 0:
        work = algorithmic(w.elem_ne[eb:eb + n], w.elem_nf[eb:eb + n])
        peaks = measured_peaks()
        hbm = peaks.get("hbm_gbs")
        cond_tflops = work["condense_flops"] / (cond_ms * 1e-3) / 1e12
        cond_gbs = work["condense_bytes"] / (cond_ms * 1e-3) / 1e9
        fp64_peak = dmma_peak or 37.2
        # the kernel hdg_plan picks for the workload's degree buckets (api.cu dispatch)
        kname = {"C1": "warp_kernel (condense_warp.cu)", "C2": "warp_kernel (condense_warp.cu)",
                 "C3": "condense_kernel, panel (condense.cu)", "C4": "sweep_kernel (condense_sweep.cu)",
                 "C5": "sweep_kernel GT/shared + condense_kernel per hp bucket (hdg_condense)"}.get(
                     args.config, "hdg_condense")
        t_fp = work["condense_flops"] / (fp64_peak * 1e12)
        t_hbm = work["condense_bytes"] / ((hbm or 6551.4) * 1e9)
        if t_fp >= t_hbm:
            roof = {"bound": "tensor", "achieved": cond_tflops, "peak": fp64_peak, "unit": "TFLOP/s",
                    "frac": cond_tflops / fp64_peak, "traffic": None,
                    "kernel": kname, "dtype": "f64 (DMMA m8n8k4 + DFMA)",
                    "peak_source": ("FP64 DMMA peak measured in this run by tools/peaks (K9)" if dmma_peak else
                                    "nominal 148 SM x 64 FP64 FMA/clk x 1.965 GHz (no in-run measurement)"),
                    "flops_per_launch": work["condense_flops"],
                    "hbm_achieved_gbs": cond_gbs, "hbm_frac": cond_gbs / (hbm or 6551.4)}
        else:
            roof = {"bound": "hbm", "achieved": cond_gbs, "peak": hbm or 6551.4, "unit": "GB/s",
                    "frac": cond_gbs / (hbm or 6551.4), "traffic": None, "kernel": kname,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if hbm else "fallback 6551.4",
                    "bytes_per_launch": work["condense_bytes"], "fp64_tflops": cond_tflops}
        # (the stored capture is of the config's default kernel: none for another degree or a forced kernel)
        default_kernel = args.degree is None and not os.environ.get("HDG_CONDENSE_KERNEL")
        roof["traffic"] = _traffic(args.config) if default_kernel else None
        line = {
            "metric": METRIC, "value": elems / (ms_step * 1e-3), "unit": "elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Philox blocks with BASELINE.json distributions, generated in HBM)",
            "config": {"workload": workload, "elements": elems, "n_e": int(w.elem_ne[eb:eb + n].max()),
                       "n_f": int(w.elem_nf[eb:eb + n].max()), "faces": w.F, "trace_dofs": w.n_trace,
                       "parallelism": f"element slabs x{world}" + (" + NCCL shared-face exchange inside "
                                                                   "hdg_assemble_skeleton" if world > 1 else ""),
                       "l2": ("inputs (%.1f GB/rank) exceed the 126 MB L2; no flush needed" % (in_bytes / 1e9)
                              if flush is None else
                              "inputs (%.3f GB/rank) under 4x the 126 MB L2: a 512 MB buffer is written before every timed step, "
                              "steps timed alone (per-step events)" % (in_bytes / 1e9)),
                       "step": "condense + assemble_skeleton + backsubstitute"},
            "condense_per_s": elems / (cond_ms * 1e-3), "backsub_per_s": elems / (bs_ms * 1e-3),
            "condense_ms": cond_ms, "assemble_ms": asm_ms, "backsub_ms": bs_ms,
            "backsub_hbm_gbs": work["backsub_bytes"] / (bs_ms * 1e-3) / 1e9,
            **({"path": "saved",
                "backsub_saved_bytes": float(sum(8 * int(a) * (int(b) + 1) + 8 * int(b) + 8 * int(a) for a, b in
                                                 zip(w.elem_ne[eb:eb + n], w.elem_nf[eb:eb + n]))),
                "note": "condense_ms is hdg_condense_saved (X written by the warp/panel kernels, a save pass on "
                        "the factors for sweep buckets); backsub_ms is the GEMV on the saved X (backsub_saved_bytes: "
                        "X, lambda_e gather, u)"} if args.path == "saved" else {}),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            **({"cuda_graph": graph} if graph else {}),
            "clocks": clk,
            "fp64_peak_tflops": {"dmma": dmma_peak, "dfma": dfma_peak},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
