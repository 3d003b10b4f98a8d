"""§8(f) NEXT #3: the skeleton solve on the GPU (block-CSR SpMV + block-Jacobi GMRES) against
the oracle: SpMV against the oracle's dense expansion of its own K; lambda against the O5 dense solve (lambda is
unique: K lambda = E); on a larger mesh the true residual recomputed on the CPU from the oracle's K."""
import numpy as np
import pytest

import gen
import oracle
from gpu_helpers import rel_fro_per_element, run_gpu, to_dev

pytestmark = pytest.mark.gpu


def _scipy_K(ref, w):
    import scipy.sparse as sp
    rp, ci, bo = ref["sym"]
    rows, cols, vals = [], [], []
    for r in range(len(rp) - 1):
        f = r
        for q in range(rp[r], rp[r + 1]):
            c = ci[q]
            a, b = int(w.face_ndof[f]), int(w.face_ndof[c])
            blk = ref["K"][bo[q]:bo[q] + a * b].reshape(a, b)
            ii, jj = np.meshgrid(np.arange(a) + w.face_off[f], np.arange(b) + w.face_off[c], indexing="ij")
            rows.append(ii.ravel())
            cols.append(jj.ravel())
            vals.append(blk.ravel())
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(w.n_trace, w.n_trace))


@pytest.mark.parametrize("name,nr,nt", [("C1", 16, 32), ("C2", 6, 12), ("C5", 4, 10), ("C3", 3, 8)])
def test_solve_matches_dense_oracle(cuda, name, nr, nt):
    import torch
    w = gen.config(name, nr=nr, nt=nt)
    blk = gen.host_blocks(w)
    ref = oracle.pipeline(w, blk=blk)                     # lambda = O5 dense solve of the oracle's K, E
    r = run_gpu(w, blk=blk)
    ctx = r["ctx"]
    # SpMV against the oracle's dense K
    x = np.random.default_rng(5).normal(size=w.n_trace)
    y = ctx.alloc("E")
    ctx.skeleton_spmv(r["K"], to_dev(x), y)
    M = oracle.to_dense(ref["sym"], ref["K"], w.face_ndof, w.face_off)
    yr = M @ x
    torch.cuda.synchronize()
    assert np.abs(y.cpu().numpy()[:w.n_trace] - yr).max() <= 1e-13 * np.abs(yr).max()
    lam = torch.zeros(w.n_trace, dtype=torch.float64, device="cuda")
    it, rr = ctx.skeleton_solve(r["K"], r["E"], lam, rtol=1e-13, maxit=2000, restart=60)
    assert rr <= 1e-12, (it, rr)
    assert np.linalg.norm(lam.cpu().numpy() - ref["lam"]) <= 1e-10 * np.linalg.norm(ref["lam"]), it
    # the reconstruction with the GPU's lambda matches the oracle's (whole pipeline with the solve inside)
    u = ctx.alloc("u")
    ctx.backsubstitute(r["factors"], r["dev"]["B"], r["dev"]["re"], lam, u)
    torch.cuda.synchronize()
    assert rel_fro_per_element(u.cpu().numpy()[:len(ref["u"])], ref["u"], ref["off_u"]) < 1e-9


def test_solve_residual_larger_mesh(cuda):
    """C3 blocks on 32 x 48 (3072 elements, ~9e4 trace dofs): the true residual of the returned lambda, recomputed
    on the CPU from the oracle's own K and E, meets the tolerance; the solve is deterministic."""
    import torch
    w = gen.config("C3", nr=32, nt=48)
    blk = gen.host_blocks(w)
    ref = oracle.pipeline(w, blk=blk, lam=np.zeros(w.n_trace))
    r = run_gpu(w, blk=blk)
    lam = torch.zeros(w.n_trace, dtype=torch.float64, device="cuda")
    it, rr = r["ctx"].skeleton_solve(r["K"], r["E"], lam, rtol=1e-10, maxit=3000, restart=50)
    Ks = _scipy_K(ref, w)
    lr = lam.cpu().numpy()
    res = np.linalg.norm(Ks @ lr - ref["E"]) / np.linalg.norm(ref["E"])
    assert res <= 2e-10, (it, rr, res)
    lam2 = torch.zeros_like(lam)
    it2, _ = r["ctx"].skeleton_solve(r["K"], r["E"], lam2, rtol=1e-10, maxit=3000, restart=50)
    assert it2 == it and torch.equal(lam, lam2)
