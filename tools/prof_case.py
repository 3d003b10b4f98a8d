"""Profiling driver: one plan + `reps` x (condense, assemble, backsub) on a BASELINE config, optionally on a
smaller annulus (same block sizes). Used under ncu; prints per-call CUDA-event times."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
import paper_1308_3995_b200 as hdg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--nr", type=int, default=None)
ap.add_argument("--nt", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
w = gen.config(a.config, nr=a.nr, nt=a.nt)
ctx = hdg.Context(0)
info = ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
inp = {}
dne, dnf = torch.from_numpy(w.elem_ne).cuda(), torch.from_numpy(w.elem_nf).cuda()
for k in ("A", "B", "C", "D", "re", "rf"):
    inp[k] = torch.empty(int(w.off[k][-1]), dtype=torch.float64, device="cuda")
    if w.uniform:
        gen.device_blocks(w, k, inp[k])
    else:
        gen.device_blocks(w, k, inp[k], off=torch.from_numpy(w.off[k]).cuda(), dev_ne=dne, dev_nf=dnf)
lam = torch.empty(w.n_trace, dtype=torch.float64, device="cuda")
gen.device_lambda(w, lam, torch.from_numpy(w.face_ndof).cuda(), torch.from_numpy(w.face_off).cuda())
S, g, u, F, inf = ctx.alloc("S"), ctx.alloc("g"), ctx.alloc("u"), ctx.alloc("factors"), ctx.alloc("info")
K, E = ctx.alloc("K"), ctx.alloc("E")
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for r in range(a.reps):
    ev[0].record()
    ctx.condense(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], S, g, F, inf)
    ev[1].record()
    ctx.assemble_skeleton(S, g, K, E)
    ev[2].record()
    ctx.backsubstitute(F, inp["B"], inp["re"], lam, u)
    ev[3].record()
    torch.cuda.synchronize()
    print(f"rep {r}: E={w.E} condense {ev[0].elapsed_time(ev[1]):.3f} ms  assemble {ev[1].elapsed_time(ev[2]):.3f} ms"
          f"  backsub {ev[2].elapsed_time(ev[3]):.3f} ms", flush=True)
