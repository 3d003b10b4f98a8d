"""oracle — plain CPU fp64 oracle of the hybridization hot path. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs may import this
package. It shares no code with the CUDA path (``paper_1308_3995_b200``); neither imports the other. Inputs come
from ``gen`` (the seeded generator, which holds none of the method's arithmetic).

Functions and the passages they follow (PAPER.md = /root/reference/PAPER.md):

* :func:`condense`   O1-O3  S_e = D_e - C_e A_e^-1 B_e, g_e = r_f - C_e A_e^-1 r_e   (Eq.
  hybridsystem; dense LU with partial pivoting per element)
* :func:`symbolic`   O4     block-CSR structure of K: one diagonal + the neighbouring edges' blocks per row
  
* :func:`assemble`   O4     K = sum_e S_e, E = sum_e g_e, element-wise, ascending element id
* :func:`dense_solve` O5    lambda = K^-1 E (LAPACK dgesv through numpy: a library primitive for the definition)
* :func:`backsub`    O6     u_e = A_e^-1 (r_e - B_e lambda_e)   (Eq. ls)
* :func:`monolithic` O7     dense solve of the uncondensed Eq. 44

Adjoint (transposed) path — SURVEY.md §8(f) NEXT #1, PAPER.md:414-436 (§4.1 "Hybridization"):

* :func:`adjoint_condense_rhs`  g~_e = r~_f - B_e^T A_e^-T r~_e   (the element part of E~ =
  -[R^T S^T][[A B][C D]]^-T [F~; G~]; H~ = 0 gives r~_f = 0)
* :func:`adjoint_assemble`      K~ = sum_e S_e^T and E~ = sum_e g~_e ("the hybridized adjoint system matrix is also the
  transpose of the hybridized primal system matrix"; K^T Lambda~ = E~)
* :func:`adjoint_backsub`       u~_e = A_e^-T (r~_e - C_e^T lambda~_e)   (the adjoint local system)

Each solves with A_e^T by its own O1/O2 factorization of A_e^T (not the primal factors); pinned by
tests/test_oracle_adjoint.py (monolithic transposed dense solve, the transpose identity, A = I closed form).

Parity status: every function is pinned by tests/test_oracle.py (brute-force monolithic solve, A = I closed
form, symmetry, LAPACK, local residuals, probe identity, pivot forcing, counts, locality, scaling).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(verbose: bool = False) -> None:
    src = os.path.join(_HERE, "oracle.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC", "-o", _SO, src,
               "-lm"]
        subprocess.run(cmd, check=True, capture_output=not verbose)


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.oracle_lu.restype = ctypes.c_int
        L.oracle_lu.argtypes = [ctypes.c_int, P, P]
        L.oracle_lu_solve.argtypes = [ctypes.c_int, P, P, ctypes.c_int, P]
        L.oracle_condense.restype = I64
        L.oracle_condense.argtypes = [I64, P, P] + [P] * 10 + [P] * 11
        L.oracle_skeleton_symbolic.restype = I64
        L.oracle_skeleton_symbolic.argtypes = [I64, I64, P, P, P, P, P, P]
        L.oracle_assemble.argtypes = [I64, I64, I64, I64] + [P] * 13
        L.oracle_backsub.argtypes = [I64, I64] + [P] * 16
        L.oracle_monolithic_build.argtypes = [I64] + [P] * 17 + [I64, P, P]
        L.oracle_dense_solve.restype = ctypes.c_int
        L.oracle_dense_solve.argtypes = [ctypes.c_int, P, P]
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(0) if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _offsets(sizes):
    o = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(np.asarray(sizes, dtype=np.int64), out=o[1:])
    return o


# ------------------------------------------------------------------------------------------------------------
def lu(a: np.ndarray):
    """O1 on one dense matrix: returns (LU, piv, info)."""
    a = _c(a, np.float64).copy()
    n = a.shape[0]
    piv = np.zeros(n, dtype=np.int32)
    info = lib().oracle_lu(n, _p(a), _p(piv))
    return a, piv, info


def lu_solve(LU, piv, b):
    """O2: A^-1 b for b of shape (n,) or (n, k)."""
    x = _c(b, np.float64).copy()
    k = 1 if x.ndim == 1 else x.shape[1]
    lib().oracle_lu_solve(LU.shape[0], _p(_c(LU, np.float64)), _p(_c(piv, np.int32)), k, _p(x))
    return x


def condense(ne, nf, blk: dict):
    """O1-O3 over a batch. ne/nf: int arrays per element; blk: dict with A,B,C,D,re,rf and off_* (as produced by
    gen.host_blocks). Returns dict S, g, LU, piv (dense packed) with offsets off_S, off_g, off_LU, off_piv, info."""
    ne = _c(ne, np.int32)
    nf = _c(nf, np.int32)
    n = len(ne)
    a64, f64 = ne.astype(np.int64), nf.astype(np.int64)
    offS, offG, offLU, offPiv = _offsets(f64 * f64), _offsets(f64), _offsets(a64 * a64), _offsets(a64)
    S = np.empty(int(offS[-1]), dtype=np.float64)
    g = np.empty(int(offG[-1]), dtype=np.float64)
    LU = np.empty(int(offLU[-1]), dtype=np.float64)
    piv = np.empty(int(offPiv[-1]), dtype=np.int32)
    info = np.zeros(n, dtype=np.int32)
    arrs = [_c(blk[k], np.float64) for k in ("A", "B", "C", "D", "re", "rf")]
    offs = [_c(blk["off_" + k], np.int64) for k in ("A", "B", "C", "D", "re", "rf")]
    lib().oracle_condense(n, _p(ne), _p(nf), *[_p(o) for o in offs], _p(offS), _p(offG), _p(offLU), _p(offPiv),
                          *[_p(a) for a in arrs], _p(S), _p(g), _p(LU), _p(piv), _p(info))
    return dict(S=S, g=g, LU=LU, piv=piv, info=info, off_S=offS, off_g=offG, off_LU=offLU, off_piv=offPiv)


def condense_shifted(ne, nf, blk: dict, shift):
    """Re-condensation (§8(f) NEXT #4): O1-O3 of A_e + diag(shift_e) — the definition written
    out: the shift (packed like r_e) is added to a copy of each element's diagonal, then the plain condensation."""
    ne = np.asarray(ne)
    A = np.array(blk["A"], dtype=np.float64, copy=True)
    oA, oR = blk["off_A"], blk["off_re"]
    for e in range(len(ne)):
        n = int(ne[e])
        for i in range(n):
            A[oA[e] + i * n + i] += shift[oR[e] + i]
    b = dict(blk)
    b["A"] = A
    return condense(ne, nf, b)


def save_solutions(ne, nf, c: dict, blk: dict):
    """§8(f) NEXT #2: the saved local solutions X_e = A_e^-1 [B_e | r_e] (n_e x (n_f + 1) row-major,
    packed per element) by O2 on each element's saved factors. Returns (X, off_X)."""
    ne = np.asarray(ne, dtype=np.int64)
    nf = np.asarray(nf, dtype=np.int64)
    offX = _offsets(ne * (nf + 1))
    X = np.empty(int(offX[-1]))
    for e in range(len(ne)):
        n, f = int(ne[e]), int(nf[e])
        rhs = np.empty((n, f + 1))
        rhs[:, :f] = np.asarray(blk["B"][blk["off_B"][e]:blk["off_B"][e + 1]]).reshape(n, f)
        rhs[:, f] = blk["re"][blk["off_re"][e]:blk["off_re"][e + 1]]
        LU = np.asarray(c["LU"][c["off_LU"][e]:c["off_LU"][e + 1]]).reshape(n, n)
        piv = c["piv"][c["off_piv"][e]:c["off_piv"][e + 1]]
        X[offX[e]:offX[e + 1]] = lu_solve(LU, piv, rhs).ravel()
    return X, offX


def backsub_saved(elem_face, face_ndof, face_off, ne, nf, X, offX, lam, e0: int = 0):
    """Reconstruction from the saved solutions: u_e = y_e - X_e[:, :n_f] lambda_e (y_e = X_e's last column),
    lambda_e gathered in slot order as O6; the sum ascending. Returns (u, off_u)."""
    ne = np.asarray(ne, dtype=np.int64)
    offU = _offsets(ne)
    u = np.empty(int(offU[-1]))
    for l in range(len(ne)):
        n, f = int(ne[l]), int(nf[l])
        lam_e = np.concatenate([np.asarray(lam[int(face_off[q]):int(face_off[q]) + int(face_ndof[q])])
                                for q in elem_face[e0 + l] if q >= 0]) if f else np.zeros(0)
        Xe = np.asarray(X[offX[l]:offX[l + 1]]).reshape(n, f + 1)
        for i in range(n):
            acc = 0.0
            for j in range(f):
                acc = acc + Xe[i, j] * lam_e[j]
            u[offU[l] + i] = Xe[i, f] - acc
    return u, offU


def symbolic(elem_face, face_elem, face_ndof, f0: int = 0, f1: int | None = None):
    """O4 symbolic over face rows [f0, f1): (row_ptr int32, col_idx int32, blk_off int64)."""
    ef, fe, fn = _c(elem_face, np.int32), _c(face_elem, np.int32), _c(face_ndof, np.int32)
    if f1 is None:
        f1 = fe.shape[0]
    L = lib()
    nnzb = L.oracle_skeleton_symbolic(f0, f1, _p(ef), _p(fe), _p(fn), None, None, None)
    row_ptr = np.zeros(f1 - f0 + 1, dtype=np.int32)
    col_idx = np.zeros(nnzb, dtype=np.int32)
    blk_off = np.zeros(nnzb + 1, dtype=np.int64)
    L.oracle_skeleton_symbolic(f0, f1, _p(ef), _p(fe), _p(fn), _p(row_ptr), _p(col_idx), _p(blk_off))
    return row_ptr, col_idx, blk_off


def assemble(elem_face, face_ndof, face_off, nf, S, offS, g, offG, sym, f0: int = 0, f1: int | None = None,
             e0: int = 0, n: int | None = None):
    """O4 numeric: K values (row-major blocks at blk_off) and E (face_off order) over rows [f0, f1) from the
    element range [e0, e0+n) (S, g, offsets and nf local to that range)."""
    row_ptr, col_idx, blk_off = sym
    fn = _c(face_ndof, np.int32)
    fo = _c(face_off, np.int64)
    if f1 is None:
        f1 = len(fn)
    if n is None:
        n = len(nf)
    K = np.empty(int(blk_off[row_ptr[-1]]), dtype=np.float64)
    E = np.empty(int(fo[f1] - fo[f0]), dtype=np.float64)
    lib().oracle_assemble(f0, f1, e0, n, _p(_c(elem_face, np.int32)), _p(fn), _p(fo), _p(_c(nf, np.int32)),
                          _p(_c(offS, np.int64)), _p(_c(offG, np.int64)), _p(_c(S, np.float64)),
                          _p(_c(g, np.float64)), _p(_c(row_ptr, np.int32)), _p(_c(col_idx, np.int32)),
                          _p(_c(blk_off, np.int64)), _p(K), _p(E))
    return K, E


def to_dense(sym, K, face_ndof, face_off, f0: int = 0):
    """Expand block-CSR rows (starting at face f0) into a dense matrix over all trace dofs."""
    row_ptr, col_idx, blk_off = sym
    nrow = len(row_ptr) - 1
    ncol = int(face_off[-1])
    r0 = int(face_off[f0])
    M = np.zeros((int(face_off[f0 + nrow]) - r0, ncol))
    for r in range(nrow):
        f = f0 + r
        for q in range(row_ptr[r], row_ptr[r + 1]):
            c = col_idx[q]
            a, b = face_ndof[f], face_ndof[c]
            M[face_off[f] - r0:face_off[f] - r0 + a, face_off[c]:face_off[c] + b] = \
                K[blk_off[q]:blk_off[q] + a * b].reshape(a, b)
    return M


def dense_solve(M, rhs):
    """O5: lambda = K^-1 E via LAPACK (numpy.linalg.solve)."""
    return np.linalg.solve(M, rhs)


def dense_solve_lu(M, rhs):
    """O5 with the oracle's own O1/O2 (tiny meshes)."""
    M = _c(M, np.float64).copy()
    x = _c(rhs, np.float64).copy()
    info = lib().oracle_dense_solve(M.shape[0], _p(M), _p(x))
    return x, info


def backsub(elem_face, face_ndof, face_off, ne, nf, LU, offLU, piv, offPiv, B, offB, re, offRe, lam, e0: int = 0):
    """O6: u_e = A_e^-1 (r_e - B_e lambda_e) for elements [e0, e0+len(ne)); returns (u, off_u)."""
    ne = _c(ne, np.int32)
    n = len(ne)
    offU = _offsets(ne.astype(np.int64))
    u = np.empty(int(offU[-1]), dtype=np.float64)
    lib().oracle_backsub(e0, n, _p(_c(elem_face, np.int32)), _p(_c(face_ndof, np.int32)), _p(_c(face_off, np.int64)),
                         _p(ne), _p(_c(nf, np.int32)), _p(_c(offLU, np.int64)), _p(_c(offPiv, np.int64)),
                         _p(_c(offB, np.int64)), _p(_c(offRe, np.int64)), _p(offU), _p(_c(LU, np.float64)),
                         _p(_c(piv, np.int32)), _p(_c(B, np.float64)), _p(_c(re, np.float64)),
                         _p(_c(lam, np.float64)), _p(u))
    return u, offU


def monolithic_system(elem_face, face_ndof, face_off, ne, nf, blk):
    """O7: the dense uncondensed matrix of Eq. 44 and its right-hand side."""
    ne = _c(ne, np.int32)
    E = len(ne)
    N = int(ne.astype(np.int64).sum() + face_off[-1])
    M = np.empty((N, N), dtype=np.float64)
    rhs = np.empty(N, dtype=np.float64)
    lib().oracle_monolithic_build(E, _p(_c(elem_face, np.int32)), _p(_c(face_ndof, np.int32)),
                                  _p(_c(face_off, np.int64)), _p(ne), _p(_c(nf, np.int32)),
                                  *[_p(_c(blk["off_" + k], np.int64)) for k in ("A", "B", "C", "D", "re", "rf")],
                                  *[_p(_c(blk[k], np.float64)) for k in ("A", "B", "C", "D", "re", "rf")],
                                  N, _p(M), _p(rhs))
    return M, rhs


def monolithic(elem_face, face_ndof, face_off, ne, nf, blk):
    """O7: solve Eq. 44 densely with O1/O2. Returns (u concatenated over elements, lambda)."""
    M, rhs = monolithic_system(elem_face, face_ndof, face_off, ne, nf, blk)
    x, info = dense_solve_lu(M, rhs)
    assert info == 0, info
    nel = int(np.asarray(ne, dtype=np.int64).sum())
    return x[:nel], x[nel:]


# ------------------------------------------------------------------------------------------------------------
def pipeline(w, blk=None, lam=None):
    """Whole oracle path on a workload: condense -> assemble (all rows) -> [lambda] -> back-substitute.
    If lam is None, lambda is the O5 dense solve of the assembled system."""
    import gen
    if blk is None:
        blk = gen.host_blocks(w)
    c = condense(w.elem_ne, w.elem_nf, blk)
    sym = symbolic(w.elem_face, w.face_elem, w.face_ndof)
    K, E = assemble(w.elem_face, w.face_ndof, w.face_off, w.elem_nf, c["S"], c["off_S"], c["g"], c["off_g"], sym)
    if lam is None:
        lam = dense_solve(to_dense(sym, K, w.face_ndof, w.face_off), E)
    u, offU = backsub(w.elem_face, w.face_ndof, w.face_off, w.elem_ne, w.elem_nf, c["LU"], c["off_LU"], c["piv"],
                      c["off_piv"], blk["B"], blk["off_B"], blk["re"], blk["off_re"], lam)
    return dict(blk=blk, cond=c, sym=sym, K=K, E=E, lam=lam, u=u, off_u=offU)


# ------------------------------------------------------------------------------------------------------------
# Adjoint (transposed) path: PAPER.md:414-436. Plain per-element loops; A_e^-T by O1/O2 on A_e^T.
def _blk(blk, key, l, shape):
    o = int(blk["off_" + key][l])
    return np.asarray(blk[key][o:o + shape[0] * shape[1]], dtype=np.float64).reshape(shape)


def _gather(elem_face, face_ndof, face_off, e, vec):
    """lambda_e: the element's faces in slot order, each face's dofs in face_off order (as O6)."""
    out = []
    for f in elem_face[e]:
        if f >= 0:
            out.append(np.asarray(vec[int(face_off[f]):int(face_off[f]) + int(face_ndof[f])], dtype=np.float64))
    return np.concatenate(out) if out else np.zeros(0)


def adjoint_condense_rhs(ne, nf, blk, rt_e, off_rt_e, rt_f=None, off_rt_f=None):
    """g~_e = r~_f - B_e^T A_e^-T r~_e per element (r~_f = 0 when not given: H~ = 0).
    Returns (g~ packed, offsets)."""
    n = len(ne)
    offG = _offsets(np.asarray(nf, dtype=np.int64))
    g = np.empty(int(offG[-1]), dtype=np.float64)
    for l in range(n):
        a, b = int(ne[l]), int(nf[l])
        A = _blk(blk, "A", l, (a, a))
        B = _blk(blk, "B", l, (a, b))
        r = np.asarray(rt_e[int(off_rt_e[l]):int(off_rt_e[l]) + a], dtype=np.float64)
        LUt, pivt, info = lu(A.T)
        assert info == 0, (l, info)
        z = lu_solve(LUt, pivt, r)                       # A_e^-T r~_e
        rf = (np.zeros(b) if rt_f is None else
              np.asarray(rt_f[int(off_rt_f[l]):int(off_rt_f[l]) + b], dtype=np.float64))
        g[int(offG[l]):int(offG[l]) + b] = rf - B.T @ z
    return g, offG


def adjoint_assemble(elem_face, face_ndof, face_off, nf, S, offS, gt, offG, sym):
    """K~ = sum_e S_e^T, E~ = sum_e g~_e: O4 applied to the transposed element matrices."""
    St = np.empty_like(np.asarray(S, dtype=np.float64))
    for l in range(len(nf)):
        b = int(nf[l])
        o = int(offS[l])
        St[o:o + b * b] = np.asarray(S[o:o + b * b], dtype=np.float64).reshape(b, b).T.reshape(-1)
    return assemble(elem_face, face_ndof, face_off, nf, St, offS, gt, offG, sym)


def adjoint_backsub(elem_face, face_ndof, face_off, ne, nf, blk, rt_e, off_rt_e, lam_t, e0: int = 0):
    """u~_e = A_e^-T (r~_e - C_e^T lambda~_e) for elements [e0, e0 + len(ne)). Returns (u~, offsets)."""
    n = len(ne)
    offU = _offsets(np.asarray(ne, dtype=np.int64))
    u = np.empty(int(offU[-1]), dtype=np.float64)
    for l in range(n):
        a, b = int(ne[l]), int(nf[l])
        A = _blk(blk, "A", l, (a, a))
        C = _blk(blk, "C", l, (b, a))
        lam = _gather(elem_face, face_ndof, face_off, e0 + l, lam_t)
        r = np.asarray(rt_e[int(off_rt_e[l]):int(off_rt_e[l]) + a], dtype=np.float64)
        LUt, pivt, info = lu(A.T)
        assert info == 0, (l, info)
        u[int(offU[l]):int(offU[l]) + a] = lu_solve(LUt, pivt, r - C.T @ lam)
    return u, offU

