"""Task timeline of the row-tile condensation kernel (condense_rows.cu) from its clock64 stamps: CTA 0, the first
512 tasks — per task its warp, the element / row tile, and the cycles spent from claim to the end of the k loop
(bulk updates with complete U rows), to the wavefront-ready point, through the diagonal block, to the end."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("HDG_CONDENSE_KERNEL", "rows")
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1308_3995_b200 as hdg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--nr", type=int, default=32)
ap.add_argument("--nt", type=int, default=64)
ap.add_argument("--show", type=int, default=80)
a = ap.parse_args()
w = gen.config(a.config, nr=a.nr, nt=a.nt)
ctx = hdg.Context(0)
ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
inp = {k: torch.empty(int(w.off[k][-1]), dtype=torch.float64, device="cuda") for k in ("A", "B", "C", "D", "re", "rf")}
for k in inp:
    gen.device_blocks(w, k, inp[k])
S, g, F, inf = ctx.alloc("S"), ctx.alloc("g"), ctx.alloc("factors"), ctx.alloc("info")
tr = torch.zeros(512 * 8, dtype=torch.int64, device="cuda")
ctx.condense(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], S, g, F, inf)
ctx.debug_set_trace(tr)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
ctx.condense(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], S, g, F, inf)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1])
t = tr.cpu().numpy().reshape(512, 8)
ne, nf = int(w.elem_ne[0]), int(w.elem_nf[0])
TA = (ne + 7) // 8
NT = TA + (nf + 7) // 8
E = w.E
per_cta = (E + 147) // 148
print(f"{a.config} {a.nr}x{a.nt}: E={E}, ~{per_cta} elements per CTA, condense {ms:.3f} ms "
      f"({ms * 1e-3 * 1.965e9 / per_cta:.0f} cycles per element per SM at 1965 MHz); {NT} tasks per element")
valid = t[:, 1] > 0
t0 = t[valid, 1].min()
n = int(valid.sum())
print(" q   warp el tile  claim@    kloop  wave   diag   rest   total")
for q in range(min(n, a.show)):
    wp, c, kd, wv, dg, en = t[q, 0], t[q, 1] - t0, t[q, 2], t[q, 3], t[q, 4], t[q, 5]
    el, tile = int(t[q, 6]), int(t[q, 7])
    isA = tile < TA
    kl = kd - t[q, 1]
    if isA:
        print(f"{q:3d} {wp:4d} {el:3d} A{tile:<3d} {c:8d} {kl:7d} {wv - kd:6d} {dg - wv:6d} {en - dg:6d} {en - t[q, 1]:7d}")
    else:
        print(f"{q:3d} {wp:4d} {el:3d} C{tile - TA:<3d} {c:8d} {kl:7d} {'':6s} {'':6s} {en - kd:6d} {en - t[q, 1]:7d}")
# per-element completion times (last task end) and throughput
ends = []
for el in range(int(t[:n, 6].max())):
    sel = t[:n, 6] == el
    if sel.sum() == NT:
        ends.append(t[:n][sel, 5].max() - t0)
ends = np.array(ends)
if len(ends) > 2:
    print("element completion (cycles):", ends.tolist())
    print("steady-state cycles per element:", float(np.median(np.diff(ends))))
busy = sum(t[q, 5] - t[q, 1] for q in range(n))
span = t[:n, 5].max() - t0
print(f"warp occupancy by tasks: {busy / (12 * span):.2f} of 12 warps over {span} cycles")
