"""Cycle breakdown of hdg_condense from the kernel's clock64 stamps (CTA 0, warps 0 and 1, first elements)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1308_3995_b200 as hdg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--nr", type=int, default=16)
ap.add_argument("--nt", type=int, default=64)
a = ap.parse_args()
w = gen.config(a.config, nr=a.nr, nt=a.nt)
ctx = hdg.Context(0)
ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
inp = {k: torch.empty(int(w.off[k][-1]), dtype=torch.float64, device="cuda") for k in ("A", "B", "C", "D", "re", "rf")}
for k in inp:
    gen.device_blocks(w, k, inp[k])
S, g, F, inf = ctx.alloc("S"), ctx.alloc("g"), ctx.alloc("factors"), ctx.alloc("info")
tr = torch.zeros(4 * 256, dtype=torch.int64, device="cuda")
ctx.condense(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], S, g, F, inf)
ctx.debug_set_trace(tr)
ctx.condense(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], S, g, F, inf)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(4, 2, 128)
npan = (int(w.elem_ne[0]) + 15) // 16
names = {0: "top", 1: "A arrived", 2: "sync", 3: "phaseA done", 4: "factors written", 5: "phaseA' done",
         6: "phaseB done", 7: "end sync"}
for it in range(1, 3):
    for wp in range(2):
        s = t[it, wp]
        base = s[0]
        print(f"element-iter {it} warp {wp}: total {t[it + 1, wp, 0] - base if it < 3 else 0} cycles")
        for k in (1, 2):
            print(f"   {names[k]:16s} +{s[k] - base:8d}")
        prev = s[2]
        for p in range(npan):
            q = s[16 + 3 * p: 19 + 3 * p]
            print(f"   panel {p}: barrier1 +{q[0] - prev:6d}  step4 {q[1] - q[0]:6d}  trailing(own) {q[2] - q[1]:6d}")
            prev = q[2]
        for k in (3, 4, 5, 6, 7):
            print(f"   {names[k]:16s} +{s[k] - base:8d}  (delta {s[k] - s[k - 1]:7d})")
