"""One row-tile condensation launch on a C4-sized mesh (HDG_CONDENSE_KERNEL=rows), for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("HDG_CONDENSE_KERNEL", "rows")
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1308_3995_b200 as hdg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
nr, nt = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (16, 64)
w = gen.config(cfg, nr=nr, nt=nt)
ctx = hdg.Context(0)
ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
inp = {k: torch.empty(int(w.off[k][-1]), dtype=torch.float64, device="cuda") for k in ("A", "B", "C", "D", "re", "rf")}
for k in inp:
    gen.device_blocks(w, k, inp[k])
S, g, F, inf = ctx.alloc("S"), ctx.alloc("g"), ctx.alloc("factors"), ctx.alloc("info")
for _ in range(2):
    ctx.condense(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], S, g, F, inf)
torch.cuda.synchronize()
print("ok", cfg, w.E)
