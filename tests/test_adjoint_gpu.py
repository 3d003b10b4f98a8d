"""GPU parity of the adjoint (transposed) path — SURVEY.md §8(f) NEXT #1, PAPER.md:414-436 — through the C ABI.

hdg_condense_adjoint_rhs (g~_e = r~_f - B_e^T A_e^-T r~_e), hdg_assemble_adjoint (K~ = sum_e S_e^T, E~ = sum g~_e)
and hdg_backsubstitute_adjoint (u~_e = A_e^-T (r~_e - C_e^T lambda~_e)) reuse the plan and the factors of the primal
hdg_condense; the oracle solves with its own factorization of A_e^T (oracle.adjoint_*). Bars as for the primal:
g~, u~ within 1e-11 relative (Frobenius, per element); the adjoint assembly of the GPU's own S bitwise equal to
the oracle's adjoint assembly of the same S; the assembled K~ equal to K^T entry by entry (the transpose identity,
SPEC.md:512, 720).
"""
import numpy as np
import pytest

import gen
import oracle
from gpu_helpers import rel_fro_per_element, run_gpu, to_dev

pytestmark = pytest.mark.gpu

TOL = 1e-11


def _adjoint_case(w, blk, with_rf=False, seed=17):
    import torch
    rng = np.random.default_rng(seed)
    rt = rng.standard_normal(int(np.sum(w.elem_ne)))
    rtf = rng.standard_normal(int(np.sum(w.elem_nf))) if with_rf else None
    lam_t = rng.standard_normal(int(w.face_off[-1]))
    r = run_gpu(w, blk=blk)
    ctx, d = r["ctx"], r["dev"]
    gt, ut = ctx.alloc("g"), ctx.alloc("u")
    Kt, Et = ctx.alloc("K"), ctx.alloc("E")
    rt_d = to_dev(rt)
    ctx.condense_adjoint_rhs(r["factors"], d["B"], rt_d, to_dev(rtf) if with_rf else None, gt)
    ctx.assemble_adjoint(r["S"], gt, Kt, Et)
    ctx.backsubstitute_adjoint(r["factors"], d["C"], rt_d, to_dev(lam_t), ut)
    torch.cuda.synchronize()
    offG = np.concatenate([[0], np.cumsum(np.asarray(w.elem_nf, dtype=np.int64))])
    g_ref, _ = oracle.adjoint_condense_rhs(w.elem_ne, w.elem_nf, blk, rt, blk["off_re"], rtf,
                                           offG if with_rf else None)
    u_ref, offU = oracle.adjoint_backsub(w.elem_face, w.face_ndof, w.face_off, w.elem_ne, w.elem_nf, blk, rt,
                                         blk["off_re"], lam_t)
    eg = rel_fro_per_element(gt.cpu().numpy()[:len(g_ref)], g_ref, offG)
    eu = rel_fro_per_element(ut.cpu().numpy()[:len(u_ref)], u_ref, offU)
    assert eg < TOL, eg
    assert eu < TOL, eu
    # adjoint assembly: bitwise against the oracle's adjoint assembly of the GPU's own S and g~; and = K^T
    S_gpu = r["S"].cpu().numpy()
    g_gpu = gt.cpu().numpy()
    offS = np.concatenate([[0], np.cumsum(np.asarray(w.elem_nf, dtype=np.int64) ** 2)])
    sym = oracle.symbolic(w.elem_face, w.face_elem, w.face_ndof)
    Kt_ref, Et_ref = oracle.adjoint_assemble(w.elem_face, w.face_ndof, w.face_off, w.elem_nf, S_gpu[:offS[-1]], offS,
                                             g_gpu[:offG[-1]], offG, sym)
    nv = len(Kt_ref)
    assert np.array_equal(Kt.cpu().numpy()[:nv], Kt_ref)
    assert np.array_equal(Et.cpu().numpy()[:len(Et_ref)], Et_ref)
    Kd = oracle.to_dense(sym, r["K"].cpu().numpy()[:nv], w.face_ndof, w.face_off)
    Ktd = oracle.to_dense(sym, Kt.cpu().numpy()[:nv], w.face_ndof, w.face_off)
    assert np.array_equal(Ktd, Kd.T)


@pytest.mark.parametrize("name,nr,nt", [("C1", 16, 32), ("C2", 4, 8), ("C3", 2, 6), ("C4", 2, 4), ("C5", 2, 6)])
def test_adjoint_parity(cuda, name, nr, nt):
    w = gen.config(name, nr=nr, nt=nt)
    _adjoint_case(w, gen.host_blocks(w))


def test_adjoint_with_rf_and_paper_boundary(cuda):
    w = gen.config("C3", nr=2, nt=5, boundary="paper")
    _adjoint_case(w, gen.host_blocks(w), with_rf=True, seed=23)


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_adjoint_pivot_forcing(cuda, name):
    """Row-permuted (A, B, r_e): the saved factors carry a non-trivial permutation, which the transposed solves
    must undo (z[perm[i]] = y[i])."""
    w = gen.config(name, nr=2, nt=4)
    blk = gen.host_blocks(w)
    rng = np.random.default_rng(29)
    for e in range(w.E):
        ne, nf = int(w.elem_ne[e]), int(w.elem_nf[e])
        A = blk["A"][blk["off_A"][e]:blk["off_A"][e + 1]].reshape(ne, ne)
        B = blk["B"][blk["off_B"][e]:blk["off_B"][e + 1]].reshape(ne, nf)
        re = blk["re"][blk["off_re"][e]:blk["off_re"][e + 1]]
        P = rng.permutation(ne)
        A[...] = A[P]
        B[...] = B[P]
        re[...] = re[P]
    _adjoint_case(w, blk, seed=31)


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_adjoint_full_size_sampled(cuda, name):
    """BASELINE.json full size in bench.py's launch configuration (bench.setup_workload, the adjoint step as
    `bench.py --path adjoint` times it): sampled elements' g~ and u~ against the oracle one by one."""
    import torch
    import bench
    wl = bench.setup_workload(name)
    w, ctx, inp, n = wl["w"], wl["ctx"], wl["inp"], wl["n"]
    ctx.condense(inp["A"], inp["B"], inp["C"], inp["D"], inp["re"], inp["rf"], wl["S"], wl["g"], wl["F"], wl["infot"])
    gt, ut = ctx.alloc("g"), ctx.alloc("u")
    ctx.condense_adjoint_rhs(wl["F"], inp["B"], inp["re"], None, gt)
    ctx.backsubstitute_adjoint(wl["F"], inp["C"], inp["re"], wl["lam"], ut)
    torch.cuda.synchronize()
    lam_t = wl["lam"].cpu().numpy()
    rng = np.random.default_rng(20261020)
    loc = np.unique(np.concatenate([np.arange(3), n - 1 - np.arange(3), rng.integers(0, n, 16)]))
    ne_l, nf_l = w.elem_ne.astype(np.int64), w.elem_nf.astype(np.int64)
    offG = np.concatenate([[0], np.cumsum(nf_l)])
    offU = np.concatenate([[0], np.cumsum(ne_l)])
    for e in loc:
        e = int(e)
        blk = gen.host_blocks(w, e, 1)
        g_ref, _ = oracle.adjoint_condense_rhs(w.elem_ne[e:e + 1], w.elem_nf[e:e + 1], blk, blk["re"], blk["off_re"])
        u_ref, _ = oracle.adjoint_backsub(w.elem_face, w.face_ndof, w.face_off, w.elem_ne[e:e + 1],
                                          w.elem_nf[e:e + 1], blk, blk["re"], blk["off_re"], lam_t, e0=e)
        g = gt[int(offG[e]):int(offG[e + 1])].cpu().numpy()
        u = ut[int(offU[e]):int(offU[e + 1])].cpu().numpy()
        assert np.linalg.norm(g - g_ref) / np.linalg.norm(g_ref) < TOL, (name, e)
        assert np.linalg.norm(u - u_ref) / np.linalg.norm(u_ref) < TOL, (name, e)


def test_adjoint_two_rank_slabs_bitwise_equal_one_rank(cuda):
    """K~ and E~ over two element slabs (emulated on one GPU): each rank assembles its owned rows from S_e^T, packs
    the S_e^T strips of shared faces for the other rank, the buffers are swapped host-side, each owner accumulates;
    the concatenated rows equal the single-rank adjoint assembly bit for bit."""
    import torch
    w = gen.config("C2", nr=4, nt=10)
    blk = gen.host_blocks(w)
    rt = np.random.default_rng(41).standard_normal(int(np.sum(w.elem_ne)))

    one = run_gpu(w, blk=blk)
    g1, K1, E1 = one["ctx"].alloc("g"), one["ctx"].alloc("K"), one["ctx"].alloc("E")
    one["ctx"].condense_adjoint_rhs(one["factors"], one["dev"]["B"], to_dev(rt), None, g1)
    one["ctx"].assemble_adjoint(one["S"], g1, K1, E1)
    reb = np.array([0, w.E // 2 - 8, w.E], dtype=np.int64)
    rs = [run_gpu(w, blk=blk, rank=r, nranks=2, rank_elem_begin=reb) for r in range(2)]
    offR = np.concatenate([[0], np.cumsum(np.asarray(w.elem_ne, dtype=np.int64))])
    outs = []
    for r in range(2):
        me = rs[r]
        rt_r = to_dev(rt[offR[reb[r]]:offR[reb[r + 1]]])
        gt, Kt, Et = me["ctx"].alloc("g"), me["ctx"].alloc("K"), me["ctx"].alloc("E")
        send = me["ctx"].alloc("send") if me["info"].send_doubles > 0 else None
        me["ctx"].condense_adjoint_rhs(me["factors"], me["dev"]["B"], rt_r, None, gt)
        me["ctx"].assemble_adjoint(me["S"], gt, Kt, Et, send=send)
        outs.append((Kt, Et, send))
    for r in range(2):
        me, other = rs[r], rs[1 - r]
        sc, sd, rc, rd = me["ctx"].exchange_counts()
        osc, osd, orc, ord_ = other["ctx"].exchange_counts()
        recv = me["ctx"].alloc("recv")
        if rc[1 - r] > 0:
            recv[rd[1 - r]:rd[1 - r] + rc[1 - r]] = outs[1 - r][2][osd[r]:osd[r] + osc[r]]
        me["ctx"].skeleton_accumulate(recv, outs[r][0], outs[r][1])
    torch.cuda.synchronize()
    K = np.concatenate([outs[r][0].cpu().numpy()[:rs[r]["info"].nvals] for r in range(2)])
    E = np.concatenate([outs[r][1].cpu().numpy()[:rs[r]["info"].n_owned_trace] for r in range(2)])
    assert np.array_equal(K, K1.cpu().numpy()[:one["info"].nvals])
    assert np.array_equal(E, E1.cpu().numpy()[:one["info"].n_owned_trace])


def test_adjoint_argument_errors(cuda):
    """No plan -> HDG_ERR_STATE; null / misaligned pointers -> HDG_ERR_ARG before anything is launched."""
    import torch
    import paper_1308_3995_b200 as hdg
    w = gen.config("C1", nr=2, nt=3)
    ctx = hdg.Context(0)
    x = torch.zeros(100000, dtype=torch.float64, device="cuda")
    F = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    with pytest.raises(hdg.HDGError) as ei:
        ctx.condense_adjoint_rhs(F, x, x, None, x)
    assert ei.value.status == hdg.HDG_ERR_STATE
    ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
    with pytest.raises(hdg.HDGError) as ei:
        ctx.condense_adjoint_rhs(F, x[1:], x, None, x)
    assert ei.value.status == hdg.HDG_ERR_ARG
    with pytest.raises(hdg.HDGError) as ei:
        ctx.condense_adjoint_rhs(F, x, x, x[1:], x)
    assert ei.value.status == hdg.HDG_ERR_ARG
    with pytest.raises(hdg.HDGError) as ei:
        ctx.backsubstitute_adjoint(F, x, x, None, x)
    assert ei.value.status == hdg.HDG_ERR_ARG
    with pytest.raises(hdg.HDGError) as ei:
        ctx.assemble_adjoint(None, x, x, x)
    assert ei.value.status == hdg.HDG_ERR_ARG


@pytest.mark.parametrize("p", [4, 5])
def test_adjoint_enriched_degree(cuda, p):
    """The adjoint at the enriched degree p + 1 ("the adjoint is approximated with p+1"): C4's
    Navier-Stokes mixed blocks at p = 4 (n_e = 180) and 5 (n_e = 252) — the elements larger than one SM, whose
    primal factors come from the global-slab sweep kernel."""
    w = gen.make_workload(f"C4-p{p}", nr=2, nt=6, m_elem=12, p_fixed=p, seed=gen.SEED_BASE + 4)
    assert int(w.elem_ne[0]) == (180 if p == 4 else 252)
    _adjoint_case(w, gen.host_blocks(w), seed=31 + p)
