"""Pins of the oracle's adjoint (transposed) path — SURVEY.md §8(f) NEXT #1.

Each check reaches the same numbers by another route: the uncondensed transposed system M^T [u~; lambda~] = [r~; 0]
solved densely (LAPACK), the transpose identity (condensing the transposed local systems gives S_e^T; the
assembled adjoint matrix is K^T entry by entry), and the A_e = I closed form.
"""
import numpy as np
import pytest

import gen
import oracle


def rel(a, b):
    d = np.linalg.norm(np.asarray(a) - np.asarray(b))
    n = np.linalg.norm(np.asarray(b))
    return d / n if n > 0 else d


def adjoint_rhs_vector(w, seed=7):
    """A seeded r~_e (packed like r_e): the functional's linearization stand-in."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal(int(np.sum(w.elem_ne)))


CASES = [("C1", 2, 4, "all"), ("C2", 2, 3, "all"), ("C3", 1, 3, "paper"), ("C5", 1, 3, "all")]


@pytest.mark.parametrize("name,nr,nt,boundary", CASES)
def test_adjoint_condensed_equals_monolithic_transposed(name, nr, nt, boundary):
    """condense the transposed system, solve K^T lambda~ = E~, reconstruct u~ — equal to the dense
    solve of the uncondensed transposed system."""
    w = gen.config(name, nr=nr, nt=nt, boundary=boundary)
    blk = gen.host_blocks(w)
    rt = adjoint_rhs_vector(w)
    c = oracle.condense(w.elem_ne, w.elem_nf, blk)
    sym = oracle.symbolic(w.elem_face, w.face_elem, w.face_ndof)
    gt, offG = oracle.adjoint_condense_rhs(w.elem_ne, w.elem_nf, blk, rt, blk["off_re"])
    Kt, Et = oracle.adjoint_assemble(w.elem_face, w.face_ndof, w.face_off, w.elem_nf, c["S"], c["off_S"], gt, offG,
                                     sym)
    lam_t = oracle.dense_solve(oracle.to_dense(sym, Kt, w.face_ndof, w.face_off), Et)
    ut, _ = oracle.adjoint_backsub(w.elem_face, w.face_ndof, w.face_off, w.elem_ne, w.elem_nf, blk, rt,
                                   blk["off_re"], lam_t)
    M, _ = oracle.monolithic_system(w.elem_face, w.face_ndof, w.face_off, w.elem_ne, w.elem_nf, blk)
    nel = int(np.sum(w.elem_ne))
    x = np.linalg.solve(M.T, np.concatenate([rt, np.zeros(M.shape[0] - nel)]))
    assert rel(ut, x[:nel]) < 1e-10
    assert rel(lam_t, x[nel:]) < 1e-10


@pytest.mark.parametrize("name,nr,nt", [("C1", 2, 4), ("C3", 1, 3), ("C5", 1, 3)])
def test_transpose_identity(name, nr, nt):
    """Condensing the transposed local systems [[A^T C^T][B^T D^T]] gives S_e^T and g~_e; the assembled adjoint
    matrix equals K^T entry by entry within 1e-12."""
    w = gen.config(name, nr=nr, nt=nt)
    blk = gen.host_blocks(w)
    rt = adjoint_rhs_vector(w, seed=11)
    c = oracle.condense(w.elem_ne, w.elem_nf, blk)
    tb = {k: np.empty_like(blk[k]) for k in ("A", "B", "C", "D")}
    tb.update({"off_A": blk["off_A"], "off_B": blk["off_B"], "off_C": blk["off_C"], "off_D": blk["off_D"],
               "re": rt, "off_re": blk["off_re"], "rf": np.zeros_like(blk["rf"]), "off_rf": blk["off_rf"]})
    for e in range(w.E):
        a, b = int(w.elem_ne[e]), int(w.elem_nf[e])
        sl = lambda k: slice(int(blk["off_" + k][e]), int(blk["off_" + k][e + 1]))
        tb["A"][sl("A")] = blk["A"][sl("A")].reshape(a, a).T.ravel()
        tb["B"][sl("B")] = blk["C"][sl("C")].reshape(b, a).T.ravel()    # (n_e x n_f) <- C_e^T
        tb["C"][sl("C")] = blk["B"][sl("B")].reshape(a, b).T.ravel()    # (n_f x n_e) <- B_e^T
        tb["D"][sl("D")] = blk["D"][sl("D")].reshape(b, b).T.ravel()
    ct = oracle.condense(w.elem_ne, w.elem_nf, tb)
    for e in range(w.E):
        b = int(w.elem_nf[e])
        S = c["S"][c["off_S"][e]:c["off_S"][e + 1]].reshape(b, b)
        St = ct["S"][ct["off_S"][e]:ct["off_S"][e + 1]].reshape(b, b)
        assert rel(St, S.T) < 1e-12
    gt, _ = oracle.adjoint_condense_rhs(w.elem_ne, w.elem_nf, blk, rt, blk["off_re"])
    assert rel(gt, ct["g"]) < 1e-12
    sym = oracle.symbolic(w.elem_face, w.face_elem, w.face_ndof)
    K, _ = oracle.assemble(w.elem_face, w.face_ndof, w.face_off, w.elem_nf, c["S"], c["off_S"], c["g"], c["off_g"],
                           sym)
    Kt, _ = oracle.adjoint_assemble(w.elem_face, w.face_ndof, w.face_off, w.elem_nf, c["S"], c["off_S"], gt,
                                    c["off_g"], sym)
    Kd = oracle.to_dense(sym, K, w.face_ndof, w.face_off)
    Ktd = oracle.to_dense(sym, Kt, w.face_ndof, w.face_off)
    assert np.abs(Ktd - Kd.T).max() <= 1e-12 * np.abs(Kd).max()


def test_identity_closed_form():
    """A_e = I: g~_e = r~_f - B_e^T r~_e and u~_e = r~_e - C_e^T lambda~_e exactly."""
    w = gen.config("C1", nr=2, nt=3)
    blk = gen.host_blocks(w)
    for e in range(w.E):
        a = int(w.elem_ne[e])
        blk["A"][blk["off_A"][e]:blk["off_A"][e + 1]] = np.eye(a).ravel()
    rt = adjoint_rhs_vector(w, seed=3)
    gt, offG = oracle.adjoint_condense_rhs(w.elem_ne, w.elem_nf, blk, rt, blk["off_re"], blk["rf"], blk["off_rf"])
    lam = np.random.default_rng(5).standard_normal(int(w.face_off[-1]))
    ut, offU = oracle.adjoint_backsub(w.elem_face, w.face_ndof, w.face_off, w.elem_ne, w.elem_nf, blk, rt,
                                      blk["off_re"], lam)
    for e in range(w.E):
        a, b = int(w.elem_ne[e]), int(w.elem_nf[e])
        B = blk["B"][blk["off_B"][e]:blk["off_B"][e + 1]].reshape(a, b)
        C = blk["C"][blk["off_C"][e]:blk["off_C"][e + 1]].reshape(b, a)
        r = rt[blk["off_re"][e]:blk["off_re"][e + 1]]
        rf = blk["rf"][blk["off_rf"][e]:blk["off_rf"][e + 1]]
        lam_e = np.concatenate([lam[w.face_off[f]:w.face_off[f] + w.face_ndof[f]] for f in w.elem_face[e] if f >= 0])
        assert np.allclose(gt[offG[e]:offG[e + 1]], rf - B.T @ r, rtol=0, atol=1e-13 * (1 + np.abs(B).sum()))
        assert np.allclose(ut[offU[e]:offU[e + 1]], r - C.T @ lam_e, rtol=0, atol=1e-13 * (1 + np.abs(C).sum()))
