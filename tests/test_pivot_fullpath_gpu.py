"""GPU parity of the pivoting and singular-element paths at the sizes where every condensation kernel runs its
full pipelined loop: each persistent CTA (or warp) condenses >= 3 elements, so an element that fails the
speculative GEPP check (R16) is redone on the exact path while the next element's loads are in flight,
clean and violating elements follow each other inside one CTA, and a violation can straddle an element boundary.

Inputs: the seeded blocks with, for a random half of the elements, the rows of (A_e, B_e, r_e) permuted (P9:
GEPP must interchange rows; S, g, u are unchanged by the permutation), a tiny leading entry in some, and a few
singular elements (one zero column of A_e: the oracle's GEPP reports info = k+1 at that column).
Every element's S, g, u is compared with the oracle at 1e-11 (S9 metric), info exactly, singular elements' S and
g must be NaN, and K/E are compared block by block where the oracle's blocks are finite (NaN pattern equal).
"""
import numpy as np
import pytest

import gen
import oracle
from gpu_helpers import run_gpu

pytestmark = pytest.mark.gpu

TOL = 1e-11


def perturb(w, blk, seed, frac=0.5, n_singular=6):
    rng = np.random.default_rng(seed)
    sing = set(rng.choice(w.E, size=min(n_singular, w.E), replace=False).tolist())
    for e in range(w.E):
        ne, nf = int(w.elem_ne[e]), int(w.elem_nf[e])
        A = blk["A"][blk["off_A"][e]:blk["off_A"][e + 1]].reshape(ne, ne)
        B = blk["B"][blk["off_B"][e]:blk["off_B"][e + 1]].reshape(ne, nf)
        re = blk["re"][blk["off_re"][e]:blk["off_re"][e + 1]]
        if rng.random() < frac:
            P = rng.permutation(ne)
            A[...] = A[P]
            B[...] = B[P]
            re[...] = re[P]
            if rng.random() < 0.2:
                A[0, 0] = 1e-13          # tiny leading entry
        if e in sing:
            A[:, int(rng.integers(0, ne))] = 0.0
    return sorted(sing)


def rel(a, b):
    n = np.linalg.norm(b)
    d = np.linalg.norm(a - b)
    return d / n if n > 0 else d


def check_perturbed(w, seed):
    blk = gen.host_blocks(w)
    sing = perturb(w, blk, seed)
    lam = gen.host_lambda(w)
    ref = oracle.pipeline(w, blk=blk, lam=lam)
    c = ref["cond"]
    r = run_gpu(w, blk=blk, lam=lam)
    info = r["infot"].cpu().numpy()[:w.E]
    assert np.array_equal(info, c["info"]), (np.nonzero(info != c["info"])[0][:10])
    assert set(np.nonzero(c["info"])[0].tolist()) == set(sing)
    S, g, u = r["S"].cpu().numpy(), r["g"].cpu().numpy(), r["u"].cpu().numpy()
    oS, og, ou = c["off_S"], c["off_g"], ref["off_u"]
    worst = {"S": 0.0, "g": 0.0, "u": 0.0}
    for e in range(w.E):
        if info[e]:
            assert np.isnan(S[oS[e]:oS[e + 1]]).all() and np.isnan(g[og[e]:og[e + 1]]).all(), e
            continue
        worst["S"] = max(worst["S"], rel(S[oS[e]:oS[e + 1]], c["S"][oS[e]:oS[e + 1]]))
        worst["g"] = max(worst["g"], rel(g[og[e]:og[e + 1]], c["g"][og[e]:og[e + 1]]))
        worst["u"] = max(worst["u"], rel(u[ou[e]:ou[e + 1]], ref["u"][ou[e]:ou[e + 1]]))
    assert all(v < TOL for v in worst.values()), worst
    K, Kref = r["K"].cpu().numpy(), ref["K"]
    bo = ref["sym"][2]
    for q in range(len(bo) - 1):
        a, b = K[bo[q]:bo[q + 1]], Kref[bo[q]:bo[q + 1]]
        assert np.array_equal(np.isnan(a), np.isnan(b)), q
        if np.isfinite(b).all():
            assert rel(a, b) < 1e-12, q
    first = r["ctx"].first_error(r["infot"])
    assert first == ((sing[0], int(c["info"][sing[0]])) if sing else (-1, 0))
    return worst


@pytest.fixture(params=["default", "sweep", "panel"])
def kernel(request, monkeypatch):
    if request.param != "default":
        monkeypatch.setenv("HDG_CONDENSE_KERNEL", request.param)
    return request.param


def test_c4_sized_480_elements(cuda, kernel):
    """n_e = 120, n_f = 48 (C4 blocks): 480 elements -> >= 3 per CTA of the one-CTA-per-SM grid."""
    w = gen.make_workload("C4", nr=10, nt=24, m_elem=12, p_fixed=3, seed=gen.SEED_BASE + 4)
    assert w.E >= 3 * 148
    check_perturbed(w, seed=401)


def test_c3_sized_900_elements(cuda, kernel):
    """n_e = 60, n_f = 60 (C3 blocks): 900 elements -> >= 3 per CTA at two CTAs per SM."""
    w = gen.make_workload("C3", nr=15, nt=30, m_elem=4, p_fixed=4, seed=gen.SEED_BASE + 3)
    assert w.E >= 3 * 296
    check_perturbed(w, seed=301)


@pytest.mark.parametrize("p", [4, 5])
def test_gt_sweep_p4_p5_480_elements(cuda, p):
    """NS p = 4 (n_e = 180, n_f = 60) and p = 5 (n_e = 252, n_f = 72): the elements larger than one SM (C5's
    heavy buckets, the sweep kernel on a global working slab), 480 elements -> >= 3 per CTA."""
    w = gen.make_workload(f"NSp{p}", nr=10, nt=24, m_elem=12, p_fixed=p, seed=gen.SEED_BASE + 5)
    assert int(w.elem_ne[0]) == (180 if p == 4 else 252)
    check_perturbed(w, seed=500 + p)


def test_ns_p2_sweep_960_elements(cuda):
    """NS p = 2 (n_e = 72, n_f = 36: C5's n_e = 72 buckets, on the shared-memory sweep kernel since session 4 of
    round 2, two CTAs per SM when they fit): 960 elements -> >= 3 per CTA."""
    w = gen.make_workload("NSp2", nr=20, nt=24, m_elem=12, p_fixed=2, seed=gen.SEED_BASE + 6)
    assert int(w.elem_ne[0]) == 72 and w.E >= 3 * 296
    check_perturbed(w, seed=602)


def test_c2_sized_7200_elements(cuda):
    """n_e = 24, n_f = 36 (C2 blocks, the warp-per-element kernel): 7200 elements -> >= 3 per warp slot at 16
    warps per SM."""
    w = gen.make_workload("C2", nr=60, nt=60, m_elem=4, p_fixed=2, seed=gen.SEED_BASE + 2)
    assert w.E >= 3 * 148 * 16
    check_perturbed(w, seed=201)


def test_hp_mesh_mixed_buckets(cuda):
    """configs[4]'s hp draw on a 12 x 40 annulus: every (n_e, n_f) bucket with permuted and singular elements."""
    w = gen.config("C5", nr=12, nt=40)
    check_perturbed(w, seed=601)
