"""Cycle breakdown of the sweep condensation kernel from its clock64 stamps (CTA 0, warp 0 = chain warp,
warp 1 = a worker, element-iterations 1..2)."""
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
for it in (1, 2):
    for wp, name in ((0, "chain warp 0"), (1, "worker warp 1")):
        s = t[it, wp]
        b = s[0]
        print(f"element-iter {it} {name}: element total {t[it + 1, wp, 0] - b} cycles")
        print(f"   D/rf loaded +{s[4] - b}  A0 landed +{s[5] - b}  all loads +{s[3] - b}")
        prev = s[3]
        for p in range(npan):
            q = s[8 + 4 * p: 12 + 4 * p]
            lbl = ("trsm4+arrive", "D-update", "diag") if wp == 0 else ("trsm", "S|g acc", "trailing")
            print(f"   panel {p}: barrier +{q[0] - prev:6d} | {lbl[0]} {q[1] - q[0]:6d} | {lbl[1]} {q[2] - q[1]:6d} | "
                  f"{lbl[2]} {q[3] - q[2]:6d}")
            prev = q[3]
        print(f"   after loop +{s[100] - prev}  ->E {s[6] - s[100]}  E wait {s[7] - s[6]}  ->end {s[101] - s[7]}")
        print(f"   reached the first panel barrier at +{s[110] - b}" + (f" (helper warp: +{t[it, 0, 112] - t[it, 1, 0]})" if wp == 1 else ""))
