"""Test-side helpers: run the libhdg path on a gen.Workload and compare with the oracle (SURVEY.md S9 metric)."""
from __future__ import annotations

import numpy as np

import gen


def rel_fro_per_element(x, ref, off):
    """max_e ||x_e - ref_e||_F / ||ref_e||_F (absolute when ||ref_e|| = 0) — SURVEY.md S9."""
    worst = 0.0
    for e in range(len(off) - 1):
        a, b = x[off[e]:off[e + 1]], ref[off[e]:off[e + 1]]
        n = np.linalg.norm(b)
        d = np.linalg.norm(a - b)
        worst = max(worst, d / n if n > 0 else d)
    return worst


def rel_per_block(K, Kref, blk_off):
    worst = 0.0
    for q in range(len(blk_off) - 1):
        a, b = K[blk_off[q]:blk_off[q + 1]], Kref[blk_off[q]:blk_off[q + 1]]
        n = np.linalg.norm(b)
        d = np.linalg.norm(a - b)
        worst = max(worst, d / n if n > 0 else d)
    return worst


def to_dev(a, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def run_gpu(w: gen.Workload, blk=None, lam=None, rank=0, nranks=1, rank_elem_begin=None, ctx=None):
    """Whole GPU path for the (slab of the) workload; returns numpy results + the context."""
    import torch
    import paper_1308_3995_b200 as hdg
    if blk is None:
        blk = gen.host_blocks(w)
    eb, n = 0, w.E
    if rank_elem_begin is not None:
        eb, n = int(rank_elem_begin[rank]), int(rank_elem_begin[rank + 1] - rank_elem_begin[rank])
    if ctx is None:
        ctx = hdg.Context(0, rank, nranks)
    info = ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne, eb, n, rank_elem_begin)
    sl = {k: blk[k][blk["off_" + k][eb]:blk["off_" + k][eb + n]] for k in ("A", "B", "C", "D", "re", "rf")}
    d = {k: to_dev(v if len(v) else np.zeros(2)) for k, v in sl.items()}
    S, g, u = ctx.alloc("S"), ctx.alloc("g"), ctx.alloc("u")
    F, infot = ctx.alloc("factors"), ctx.alloc("info")
    ctx.condense(d["A"], d["B"], d["C"], d["D"], d["re"], d["rf"], S, g, F, infot)
    K, E = ctx.alloc("K"), ctx.alloc("E")
    rp, ci, bo = ctx.alloc("row_ptr"), ctx.alloc("col_idx"), ctx.alloc("blk_off")
    send = ctx.alloc("send") if info.send_doubles > 0 else None
    ctx.assemble_skeleton(S, g, K, E, rp, ci, bo, send)
    out = dict(ctx=ctx, info=info, S=S, g=g, K=K, E=E, row_ptr=rp, col_idx=ci, blk_off=bo, factors=F, infot=infot,
               send=send, dev=d)
    if lam is not None:
        lt = to_dev(lam)
        ctx.backsubstitute(F, d["B"], d["re"], lt, u)
        out["u"] = u
    torch.cuda.synchronize()
    return out


def np_out(r, key, n=None):
    t = r[key]
    a = t.cpu().numpy()
    return a if n is None else a[:n]
