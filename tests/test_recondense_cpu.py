"""§8(f) NEXT #4 on the CPU: the re-condensation oracle with the pseudo-time shift pinned to
closed forms, and the DG-vs-HDG nonzero counts (Tables 1-4; SPEC.md dg_nnz) of libhdg's host-only
hdg_nnz_counts pinned to SPEC's worked examples and to an assemble-and-count brute force."""
import numpy as np
import pytest

import gen
import oracle


def _blk_single(ne, nf, A, B, C, D, re, rf):
    return dict(A=A.ravel().copy(), B=B.ravel().copy(), C=C.ravel().copy(), D=D.ravel().copy(), re=re.copy(),
                rf=rf.copy(), off_A=np.array([0, ne * ne]), off_B=np.array([0, ne * nf]),
                off_C=np.array([0, nf * ne]), off_D=np.array([0, nf * nf]), off_re=np.array([0, ne]),
                off_rf=np.array([0, nf]))


def test_shift_on_zero_matrix_closed_form():
    """A_e = 0 plus a uniform shift sigma: A_e + diag(s) = sigma I, so S = D - C B / sigma, g = r_f - C r_e / sigma
    (a dropped shift, a shift off the diagonal or a wrong index fails this)."""
    rng = np.random.default_rng(3)
    ne, nf, sigma = 12, 24, 2.5
    B, C, D = rng.normal(size=(ne, nf)), rng.normal(size=(nf, ne)), rng.normal(size=(nf, nf))
    re, rf = rng.normal(size=ne), rng.normal(size=nf)
    blk = _blk_single(ne, nf, np.zeros((ne, ne)), B, C, D, re, rf)
    c = oracle.condense_shifted([ne], [nf], blk, np.full(ne, sigma))
    S = c["S"].reshape(nf, nf)
    assert np.abs(S - (D - C @ B / sigma)).max() <= 1e-14 * np.abs(D).max()
    assert np.abs(c["g"] - (rf - C @ re / sigma)).max() <= 1e-14 * np.abs(rf).max()


def test_shift_large_sigma_asymptotics():
    """dt -> 0 (sigma -> inf): S = D - C (A + sigma I)^-1 B = D - C B / sigma + C A B / sigma^2 + O(sigma^-3)."""
    rng = np.random.default_rng(4)
    ne, nf, sigma = 24, 36, 1e4
    A, B, C, D = (rng.normal(size=s) for s in ((ne, ne), (ne, nf), (nf, ne), (nf, nf)))
    blk = _blk_single(ne, nf, A, B, C, D, rng.normal(size=ne), rng.normal(size=nf))
    S = oracle.condense_shifted([ne], [nf], blk, np.full(ne, sigma))["S"].reshape(nf, nf)
    approx = D - C @ B / sigma + C @ A @ B / sigma ** 2
    assert np.abs(S - approx).max() <= 10 * np.abs(C @ A @ A @ B).max() / sigma ** 3 + 1e-13


def test_zero_shift_is_plain_condensation():
    w = gen.config("C2", nr=2, nt=3)
    blk = gen.host_blocks(w)
    a = oracle.condense(w.elem_ne, w.elem_nf, blk)
    b = oracle.condense_shifted(w.elem_ne, w.elem_nf, blk, np.zeros(int(w.off["re"][-1])))
    assert np.array_equal(a["S"], b["S"]) and np.array_equal(a["g"], b["g"])


def test_pseudo_time_shift_structure():
    """Shift on the w unknowns only ([Q; W] basis-major, DESIGN R4), positive, scaling as 1 / CFL."""
    w = gen.config("C4", nr=2, nt=3)
    s1 = gen.pseudo_time_shift(w, 1.0)
    s2 = gen.pseudo_time_shift(w, 4.0)
    assert np.allclose(s1, 4.0 * s2)
    ne = int(w.elem_ne[0])
    nw = 4 * ne // 12
    for e in range(w.E):
        blk = s1[e * ne:(e + 1) * ne]
        assert (blk[:ne - nw] == 0).all() and (blk[ne - nw:] > 1.0).all() and len(set(blk[ne - nw:])) == 1
    assert gen.cfl_ramp(0) == 0.0 and gen.cfl_ramp(10) == pytest.approx(10.0)
    assert all(gen.cfl_ramp(n) < gen.cfl_ramp(n + 1) for n in range(10))


# ---- DG vs HDG nonzeros --------------------------------------------------------------------------------------
def _mesh_one():
    ef = np.array([[0, 1, 2]], dtype=np.int32)
    fe = np.array([[0, -1], [0, -1], [0, -1]], dtype=np.int32)
    return ef, fe


def _mesh_two():
    ef = np.array([[0, 1, 2], [2, 3, 4]], dtype=np.int32)
    fe = np.array([[0, -1], [0, -1], [0, 1], [1, -1], [1, -1]], dtype=np.int32)
    return ef, fe


def test_nnz_spec_examples():
    import paper_1308_3995_b200 as hdg
    ef, fe = _mesh_one()
    dg, _ = hdg.nnz_counts(ef, fe, np.full(3, 2, dtype=np.int32), np.array([3], dtype=np.int32))
    assert dg == 9                      # 1 element, p = 1, m = 1: n(1)^2
    ef, fe = _mesh_two()
    dg, hdgn = hdg.nnz_counts(ef, fe, np.full(5, 2, dtype=np.int32), np.array([3, 3], dtype=np.int32))
    assert dg == 9 + 9 + 2 * 9          # 2 elements sharing an edge
    # HDG rows: faces 0, 1 see 3 faces each, face 2 sees all 5, faces 3, 4 see 3 each; 2 dofs per face
    assert hdgn == 4 * (3 + 3 + 5 + 3 + 3)


def _brute_dg(w, d):
    off = np.concatenate([[0], np.cumsum(d)])
    M = np.zeros((off[-1], off[-1]), dtype=bool)
    for e in range(w.E):
        M[off[e]:off[e + 1], off[e]:off[e + 1]] = True
    for l, r in w.face_elem:
        if r >= 0:
            M[off[l]:off[l + 1], off[r]:off[r + 1]] = True
            M[off[r]:off[r + 1], off[l]:off[l + 1]] = True
    return int(M.sum())


@pytest.mark.parametrize("name", ["C1", "C5"])
def test_nnz_against_assemble_and_count(name):
    import paper_1308_3995_b200 as hdg
    w = gen.config(name, nr=3, nt=5)
    d = (4 * gen.n_modes(w.p)).astype(np.int32)            # DG: m = 4 equations, n(p_K) modes
    dg, hdgn = hdg.nnz_counts(w.elem_face, w.face_elem, w.face_ndof, d)
    assert dg == _brute_dg(w, d)
    assert hdgn == int(oracle.symbolic(w.elem_face, w.face_elem, w.face_ndof)[2][-1])


def test_nnz_ratio_grows_with_p():
    """'the ratio grows with increasing polynomial degree in favor of HDG' on a fixed mesh
    (paper boundary mode: Gamma_h only)."""
    import paper_1308_3995_b200 as hdg
    ratios = []
    for p in range(1, 6):
        w = gen.make_workload("r", nr=4, nt=8, m_elem=4, p_fixed=p, seed=1, boundary="paper")
        dg, hdgn = hdg.nnz_counts(w.elem_face, w.face_elem, w.face_ndof,
                                  (4 * gen.n_modes(w.p)).astype(np.int32))
        ratios.append(dg / hdgn)
    assert all(a < b for a, b in zip(ratios, ratios[1:])), ratios
