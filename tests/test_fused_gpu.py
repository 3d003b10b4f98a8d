"""§8(f) NEXT #2, fused condense -> assemble (hdg_condense_assemble): S_e and g_e go from the condensation kernels
straight into K and E. Each K / E entry has at most two contributions and (0 + a) + b = (0 + b) + a in IEEE
arithmetic, so K and E must be BITWISE those of hdg_condense + hdg_assemble_skeleton (the ordered gather) — on every
condensation kernel, with singular elements (NaN rows) and in the paper's boundary mode."""
import numpy as np
import pytest

import gen
from gpu_helpers import run_gpu, to_dev

pytestmark = pytest.mark.gpu


def _fused(w, blk):
    import torch
    import paper_1308_3995_b200 as hdg
    ctx = hdg.Context(0)
    info = ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
    d = {k: to_dev(blk[k]) for k in ("A", "B", "C", "D", "re", "rf")}
    K, E, F, inf = ctx.alloc("K"), ctx.alloc("E"), ctx.alloc("factors"), ctx.alloc("info")
    K.fill_(7.0)                      # the call zeroes K, E itself
    ctx.condense_assemble(d["A"], d["B"], d["C"], d["D"], d["re"], d["rf"], K, E, F, inf)
    rp, ci = ctx.alloc("row_ptr"), ctx.alloc("col_idx")
    ctx.skeleton_structure(rp, ci)
    torch.cuda.synchronize()
    return info, K.cpu().numpy()[:info.nvals], E.cpu().numpy()[:info.n_owned_trace], inf.cpu().numpy()[:w.E], rp, ci


@pytest.mark.parametrize("name,nr,nt,kern", [("C1", 3, 5, None), ("C2", 4, 8, None), ("C3", 3, 8, None),
                                             ("C3", 3, 8, "rows"), ("C4", 3, 6, None), ("C4", 3, 6, "panel"),
                                             ("C4", 3, 6, "rows"), ("C5", 4, 10, None)])
def test_fused_bitwise_equals_gather(cuda, monkeypatch, name, nr, nt, kern):
    if kern:
        monkeypatch.setenv("HDG_CONDENSE_KERNEL", kern)
    w = gen.config(name, nr=nr, nt=nt)
    blk = gen.host_blocks(w)
    r = run_gpu(w, blk=blk)
    info, K, E, inf, rp, ci = _fused(w, blk)
    assert np.array_equal(K, r["K"].cpu().numpy()[:info.nvals])
    assert np.array_equal(E, r["E"].cpu().numpy()[:info.n_owned_trace])
    assert np.array_equal(rp.cpu().numpy(), r["row_ptr"].cpu().numpy())
    assert (inf == 0).all()


def test_fused_singular_and_paper_boundary(cuda):
    """A singular element: its NaN S rows reach exactly the K blocks and E entries its faces touch (as in the
    gather); paper boundary mode: slots without trace carry nothing."""
    w = gen.config("C3", nr=3, nt=7, boundary="paper")
    blk = gen.host_blocks(w)
    e_bad = 9
    ne = int(w.elem_ne[e_bad])
    A = blk["A"][blk["off_A"][e_bad]:blk["off_A"][e_bad + 1]].reshape(ne, ne)
    A[:, 11] = 0.0
    r = run_gpu(w, blk=blk)
    info, K, E, inf, _, _ = _fused(w, blk)
    Kg, Eg = r["K"].cpu().numpy()[:info.nvals], r["E"].cpu().numpy()[:info.n_owned_trace]
    assert inf[e_bad] == 12
    assert np.array_equal(np.isnan(K), np.isnan(Kg)) and np.isnan(K).any()
    assert np.array_equal(K[~np.isnan(K)], Kg[~np.isnan(Kg)])
    assert np.array_equal(np.isnan(E), np.isnan(Eg))
    assert np.array_equal(E[~np.isnan(E)], Eg[~np.isnan(Eg)])


def test_fused_gt_sweep_p4(cuda):
    w = gen.make_workload("NSp4", nr=2, nt=6, m_elem=12, p_fixed=4, seed=gen.SEED_BASE + 5)
    blk = gen.host_blocks(w)
    r = run_gpu(w, blk=blk)
    info, K, E, _, _, _ = _fused(w, blk)
    assert np.array_equal(K, r["K"].cpu().numpy()[:info.nvals])
    assert np.array_equal(E, r["E"].cpu().numpy()[:info.n_owned_trace])
