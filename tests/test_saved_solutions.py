"""§8(f) NEXT #2: the saved local solutions. CPU pins of the oracle extension (the identity
A^-1 (r - B lambda) = A^-1 r - (A^-1 B) lambda against O6, and the A = I closed form X = [B | r]) and GPU parity of
hdg_save_solutions / hdg_backsubstitute_saved against it on every config's block sizes."""
import numpy as np
import pytest

import gen
import oracle
from gpu_helpers import rel_fro_per_element, to_dev


def _uvec_oracle(w, blk, lam):
    c = oracle.condense(w.elem_ne, w.elem_nf, blk)
    X, offX = oracle.save_solutions(w.elem_ne, w.elem_nf, c, blk)
    us, offU = oracle.backsub_saved(w.elem_face, w.face_ndof, w.face_off, w.elem_ne, w.elem_nf, X, offX, lam)
    return c, X, offX, us, offU


@pytest.mark.parametrize("name", ["C1", "C4", "C5"])
def test_saved_reconstruction_equals_O6(name):
    w = gen.config(name, nr=2, nt=3)
    blk = gen.host_blocks(w)
    lam = gen.host_lambda(w)
    c, X, offX, us, offU = _uvec_oracle(w, blk, lam)
    u, offU2 = oracle.backsub(w.elem_face, w.face_ndof, w.face_off, w.elem_ne, w.elem_nf, c["LU"], c["off_LU"],
                              c["piv"], c["off_piv"], blk["B"], blk["off_B"], blk["re"], blk["off_re"], lam)
    assert np.array_equal(offU, offU2)
    assert rel_fro_per_element(us, u, offU) < 1e-13


def test_saved_solutions_identity_closed_form():
    """A_e = I: X_e = [B_e | r_e] exactly."""
    w = gen.config("C2", nr=2, nt=3)
    blk = gen.host_blocks(w)
    for e in range(w.E):
        n = int(w.elem_ne[e])
        blk["A"][blk["off_A"][e]:blk["off_A"][e + 1]] = np.eye(n).ravel()
    c = oracle.condense(w.elem_ne, w.elem_nf, blk)
    X, offX = oracle.save_solutions(w.elem_ne, w.elem_nf, c, blk)
    for e in range(w.E):
        n, f = int(w.elem_ne[e]), int(w.elem_nf[e])
        Xe = X[offX[e]:offX[e + 1]].reshape(n, f + 1)
        assert np.array_equal(Xe[:, :f], blk["B"][blk["off_B"][e]:blk["off_B"][e + 1]].reshape(n, f))
        assert np.array_equal(Xe[:, f], blk["re"][blk["off_re"][e]:blk["off_re"][e + 1]])


@pytest.mark.gpu
@pytest.mark.parametrize("name,nr,nt", [("C1", 3, 5), ("C2", 4, 8), ("C3", 3, 8), ("C4", 3, 6), ("C5", 4, 10)])
def test_saved_solutions_gpu(cuda, name, nr, nt):
    import torch
    import paper_1308_3995_b200 as hdg
    w = gen.config(name, nr=nr, nt=nt)
    blk = gen.host_blocks(w)
    lam = gen.host_lambda(w)
    c, X, offX, us, offU = _uvec_oracle(w, blk, lam)
    ctx = hdg.Context(0)
    info = ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
    assert info.len_X == len(X)
    d = {k: to_dev(blk[k]) for k in ("A", "B", "C", "D", "re", "rf")}
    S, g, F, inf = ctx.alloc("S"), ctx.alloc("g"), ctx.alloc("factors"), ctx.alloc("info")
    ctx.condense(d["A"], d["B"], d["C"], d["D"], d["re"], d["rf"], S, g, F, inf)
    Xg, u = ctx.alloc("X"), ctx.alloc("u")
    ctx.save_solutions(F, d["B"], d["re"], Xg)
    ctx.backsubstitute_saved(Xg, to_dev(lam), u)
    torch.cuda.synchronize()
    assert rel_fro_per_element(Xg.cpu().numpy()[:len(X)], X, offX) < 1e-11
    assert rel_fro_per_element(u.cpu().numpy()[:len(us)], us, offU) < 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("name,nr,nt,kern", [("C2", 4, 8, None), ("C3", 3, 8, None), ("C3", 3, 8, "sweep"),
                                             ("C4", 3, 6, None), ("C4", 3, 6, "panel"), ("C5", 4, 10, None)])
def test_condense_saved_fused(cuda, monkeypatch, name, nr, nt, kern):
    """hdg_condense_saved: X written by the warp / panel kernels during the condensation, by the save pass for the
    sweep buckets — the same X as the oracle's, and the same S, g as hdg_condense."""
    import torch
    import paper_1308_3995_b200 as hdg
    if kern:
        monkeypatch.setenv("HDG_CONDENSE_KERNEL", kern)
    w = gen.config(name, nr=nr, nt=nt)
    blk = gen.host_blocks(w)
    lam = gen.host_lambda(w)
    c, X, offX, us, offU = _uvec_oracle(w, blk, lam)
    ctx = hdg.Context(0)
    ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
    d = {k: to_dev(blk[k]) for k in ("A", "B", "C", "D", "re", "rf")}
    S, g, F, inf, Xg, u = (ctx.alloc(k) for k in ("S", "g", "factors", "info", "X", "u"))
    ctx.condense_saved(d["A"], d["B"], d["C"], d["D"], d["re"], d["rf"], S, g, F, Xg, inf)
    ctx.backsubstitute_saved(Xg, to_dev(lam), u)
    torch.cuda.synchronize()
    assert rel_fro_per_element(Xg.cpu().numpy()[:len(X)], X, offX) < 1e-11
    assert rel_fro_per_element(S.cpu().numpy()[:len(c["S"])], c["S"], c["off_S"]) < 1e-11
    assert rel_fro_per_element(u.cpu().numpy()[:len(us)], us, offU) < 1e-11
