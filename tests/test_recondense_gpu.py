"""§8(f) NEXT #4 on the GPU: hdg_condense_shifted (A_e + diag(shift_e), the pseudo-time term of PAPER.md:303-313
applied while the kernels stage A_e) against oracle.condense_shifted, on every condensation kernel, and the
back-substitution with the shifted factors; a sequence of re-condensations along the CFL ramp."""
import numpy as np
import pytest

import gen
import oracle
from gpu_helpers import rel_fro_per_element, to_dev

pytestmark = pytest.mark.gpu
TOL = 1e-11


def run_shifted(w, blk, shift, lam):
    import torch
    import paper_1308_3995_b200 as hdg
    ctx = hdg.Context(0)
    ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
    d = {k: to_dev(blk[k]) for k in ("A", "B", "C", "D", "re", "rf")}
    S, g, u, F, inf = ctx.alloc("S"), ctx.alloc("g"), ctx.alloc("u"), ctx.alloc("factors"), ctx.alloc("info")
    ctx.condense_shifted(d["A"], d["B"], d["C"], d["D"], d["re"], d["rf"], to_dev(shift), S, g, F, inf)
    ctx.backsubstitute(F, d["B"], d["re"], to_dev(lam), u)
    torch.cuda.synchronize()
    return S.cpu().numpy(), g.cpu().numpy(), u.cpu().numpy(), inf.cpu().numpy()[:w.E]


@pytest.mark.parametrize("name,kern,nr,nt", [("C2", None, 4, 8), ("C3", None, 3, 8), ("C3", "rows", 3, 8),
                                             ("C4", None, 3, 6), ("C4", "panel", 3, 6), ("C4", "rows", 3, 6),
                                             ("C5", None, 4, 10)])
def test_shifted_condensation_matches_oracle(cuda, monkeypatch, name, kern, nr, nt):
    if kern:
        monkeypatch.setenv("HDG_CONDENSE_KERNEL", kern)
    w = gen.config(name, nr=nr, nt=nt)
    blk = gen.host_blocks(w)
    lam = gen.host_lambda(w)
    shift = gen.pseudo_time_shift(w, gen.cfl_ramp(2))
    S, g, u, info = run_shifted(w, blk, shift, lam)
    c = oracle.condense_shifted(w.elem_ne, w.elem_nf, blk, shift)
    assert (info == 0).all()
    assert rel_fro_per_element(S, c["S"], c["off_S"]) < TOL
    assert rel_fro_per_element(g, c["g"], c["off_g"]) < TOL
    ushift, offU = oracle.backsub(w.elem_face, w.face_ndof, w.face_off, w.elem_ne, w.elem_nf, c["LU"], c["off_LU"],
                                  c["piv"], c["off_piv"], blk["B"], blk["off_B"], blk["re"], blk["off_re"], lam)
    assert rel_fro_per_element(u, ushift, offU) < TOL


def test_shifted_gt_sweep_p4(cuda):
    """n_e = 180 (the global-slab sweep kernel) with the shift."""
    w = gen.make_workload("NSp4", nr=2, nt=6, m_elem=12, p_fixed=4, seed=gen.SEED_BASE + 5)
    blk = gen.host_blocks(w)
    lam = gen.host_lambda(w)
    shift = gen.pseudo_time_shift(w, 0.7)
    S, g, u, info = run_shifted(w, blk, shift, lam)
    c = oracle.condense_shifted(w.elem_ne, w.elem_nf, blk, shift)
    assert rel_fro_per_element(S, c["S"], c["off_S"]) < TOL
    assert rel_fro_per_element(g, c["g"], c["off_g"]) < TOL


def test_recondensation_along_cfl_ramp(cuda):
    """Newton steps n = 1..4 of the ramp re-condense with the changing shift; the last step with CFL -> inf is
    the plain condensation (pure Newton-Raphson)."""
    import torch
    import paper_1308_3995_b200 as hdg
    w = gen.config("C4", nr=2, nt=5)
    blk = gen.host_blocks(w)
    ctx = hdg.Context(0)
    ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
    d = {k: to_dev(blk[k]) for k in ("A", "B", "C", "D", "re", "rf")}
    S, g, F, inf = ctx.alloc("S"), ctx.alloc("g"), ctx.alloc("factors"), ctx.alloc("info")
    for n in (1, 2, 3, 4):
        shift = gen.pseudo_time_shift(w, gen.cfl_ramp(n))
        ctx.condense_shifted(d["A"], d["B"], d["C"], d["D"], d["re"], d["rf"], to_dev(shift), S, g, F, inf)
        torch.cuda.synchronize()
        c = oracle.condense_shifted(w.elem_ne, w.elem_nf, blk, shift)
        assert rel_fro_per_element(S.cpu().numpy(), c["S"], c["off_S"]) < TOL, n
    ctx.condense_shifted(d["A"], d["B"], d["C"], d["D"], d["re"], d["rf"], to_dev(np.zeros(int(w.off["re"][-1]))),
                         S, g, F, inf)
    S0, g0 = S.clone(), g.clone()
    ctx.condense(d["A"], d["B"], d["C"], d["D"], d["re"], d["rf"], S, g, F, inf)
    torch.cuda.synchronize()
    assert torch.equal(S0, S) and torch.equal(g0, g)
