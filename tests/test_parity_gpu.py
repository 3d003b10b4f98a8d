"""GPU parity: libhdg (sm_100a CUDA, through the C ABI) against the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north_star): block-CSR row_ptr/col_idx/blk_off bit-exact; S, g, u within
max relative error 1e-11 (Frobenius, per element); assembled skeleton values within 1e-12 relative per block
(and bitwise when the GPU assembles the oracle's own S, g — the left-then-right two-term sum is exact).
"""
import numpy as np
import pytest

import gen
import oracle
from gpu_helpers import rel_fro_per_element, rel_per_block, run_gpu, to_dev

pytestmark = pytest.mark.gpu

TOL = 1e-11
KTOL = 1e-12


def check_all(w, blk=None, lam=None, with_u=True):
    if blk is None:
        blk = gen.host_blocks(w)
    if lam is None:
        lam = gen.host_lambda(w)
    ref = oracle.pipeline(w, blk=blk, lam=lam)
    r = run_gpu(w, blk=blk, lam=lam if with_u else None)
    c = ref["cond"]
    assert (r["infot"].cpu().numpy()[:w.E] == 0).all()
    eS = rel_fro_per_element(r["S"].cpu().numpy(), c["S"], c["off_S"])
    eg = rel_fro_per_element(r["g"].cpu().numpy(), c["g"], c["off_g"])
    assert eS < TOL, eS
    assert eg < TOL, eg
    rp, ci, bo = ref["sym"]
    assert np.array_equal(r["row_ptr"].cpu().numpy(), rp)
    assert np.array_equal(r["col_idx"].cpu().numpy()[:len(ci)], ci)
    assert np.array_equal(r["blk_off"].cpu().numpy(), bo)
    eK = rel_per_block(r["K"].cpu().numpy(), ref["K"], bo)
    assert eK < KTOL, eK
    eE = rel_fro_per_element(r["E"].cpu().numpy(), ref["E"], w.face_off)
    assert eE < KTOL, eE
    if with_u:
        eu = rel_fro_per_element(r["u"].cpu().numpy(), ref["u"], ref["off_u"])
        assert eu < TOL, eu
    return r, ref


def test_c1_full_end_to_end(cuda):
    """C1 (BASELINE configs[0]) at full size; lambda from the oracle's dense solve of the skeleton system (O5)."""
    w = gen.config("C1")
    blk = gen.host_blocks(w)
    ref = oracle.pipeline(w, blk=blk)           # lambda = K^-1 E (O5)
    r, _ = check_all(w, blk=blk, lam=ref["lam"])
    # P7 with the GPU's u: element rows A u + B lambda = r_e, face rows sum (C u + D lambda) = sum r_f
    u = r["u"].cpu().numpy()
    lam = ref["lam"]
    face_rows = np.zeros(w.n_trace)
    rhs = np.zeros(w.n_trace)
    for e in range(w.E):
        A = blk["A"][blk["off_A"][e]:blk["off_A"][e + 1]].reshape(12, 12)
        B = blk["B"][blk["off_B"][e]:blk["off_B"][e + 1]].reshape(12, 24)
        C = blk["C"][blk["off_C"][e]:blk["off_C"][e + 1]].reshape(24, 12)
        D = blk["D"][blk["off_D"][e]:blk["off_D"][e + 1]].reshape(24, 24)
        idx = np.concatenate([np.arange(w.face_off[f], w.face_off[f + 1]) for f in w.elem_face[e]])
        ue = u[12 * e:12 * e + 12]
        res = A @ ue + B @ lam[idx] - blk["re"][12 * e:12 * e + 12]
        assert np.abs(res).max() < 1e-13 * max(1, np.abs(ue).max())
        np.add.at(face_rows, idx, C @ ue + D @ lam[idx])
        np.add.at(rhs, idx, blk["rf"][24 * e:24 * e + 24])
    assert np.abs(face_rows - rhs).max() < 1e-13 * np.abs(rhs).max()


@pytest.mark.parametrize("name,nr,nt", [("C2", 8, 16), ("C3", 6, 11), ("C4", 4, 9)])
def test_uniform_configs_reduced_mesh(cuda, name, nr, nt):
    """BASELINE configs[1..3] block sizes on meshes the oracle finishes in seconds (many tiles, ragged tails)."""
    check_all(gen.config(name, nr=nr, nt=nt))


def test_hp_config_reduced_mesh(cuda):
    """configs[4]: hp degree draw, every (n_e, n_f) bucket incl. the p >= 4 global-scratch path."""
    w = gen.config("C5", nr=6, nt=12)
    assert set(np.unique(w.p)) == {1, 2, 3, 4, 5}
    check_all(w)


@pytest.mark.parametrize("name", ["C1", "C3", "C5"])
def test_paper_boundary_mode(cuda, name):
    """Gamma_h only: ring elements have one slot without trace -> ragged n_f buckets."""
    check_all(gen.config(name, nr=3, nt=7, boundary="paper"))


@pytest.mark.parametrize("name", ["C1", "C3", "C4"])
def test_pivot_forcing(cuda, name):
    """P9: row-permuted (A, B, r_e) must give the same S, g, u; seeded inputs alone never swap rows."""
    w = gen.config(name, nr=2, nt=5)
    blk = gen.host_blocks(w)
    rng = np.random.default_rng(91)
    for e in range(w.E):
        ne, nf = int(w.elem_ne[e]), int(w.elem_nf[e])
        A = blk["A"][blk["off_A"][e]:blk["off_A"][e + 1]].reshape(ne, ne)
        B = blk["B"][blk["off_B"][e]:blk["off_B"][e + 1]].reshape(ne, nf)
        re = blk["re"][blk["off_re"][e]:blk["off_re"][e + 1]]
        P = rng.permutation(ne)
        A[...] = A[P]
        B[...] = B[P]
        re[...] = re[P]
        if e % 3 == 0:
            A[0, 0] = 1e-13      # tiny leading entry
    check_all(w, blk=blk)


def test_assembly_of_oracle_S_is_bitwise(cuda):
    """Isolated assembly: the GPU assembling the oracle's S, g reproduces the oracle's K, E bit for bit."""
    import paper_1308_3995_b200 as hdg
    w = gen.config("C5", nr=5, nt=9)
    ref = oracle.pipeline(w, lam=np.zeros(gen.config("C5", nr=5, nt=9).n_trace))
    ctx = hdg.Context(0)
    info = ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
    K, E = ctx.alloc("K"), ctx.alloc("E")
    ctx.assemble_skeleton(to_dev(ref["cond"]["S"]), to_dev(ref["cond"]["g"]), K, E)
    assert np.array_equal(K.cpu().numpy()[:info.nvals], ref["K"])
    assert np.array_equal(E.cpu().numpy()[:info.n_owned_trace], ref["E"])


def test_two_rank_slabs_bitwise_equal_one_rank(cuda):
    """P12 (emulated on one GPU, no waiting kernels): rank slabs assemble locally, pack their contributions to
    rows owned by the other rank, the buffers are swapped on the host side, and each owner accumulates. The
    concatenated owned rows equal the single-rank assembly bit for bit."""
    w = gen.config("C2", nr=4, nt=10)
    blk = gen.host_blocks(w)
    one = run_gpu(w, blk=blk)
    reb = np.array([0, w.E // 2 - 8, w.E], dtype=np.int64)   # uneven slabs
    rs = [run_gpu(w, blk=blk, rank=r, nranks=2, rank_elem_begin=reb) for r in range(2)]
    for r in range(2):
        me, other = rs[r], rs[1 - r]
        sc, sd, rc, rd = me["ctx"].exchange_counts()
        osc, osd, orc, ord_ = other["ctx"].exchange_counts()
        assert rc[1 - r] == osc[r]
        recv = me["ctx"].alloc("recv")
        if rc[1 - r] > 0:
            recv[rd[1 - r]:rd[1 - r] + rc[1 - r]] = other["send"][osd[r]:osd[r] + osc[r]]
        me["ctx"].skeleton_accumulate(recv, me["K"], me["E"])
    import torch
    torch.cuda.synchronize()
    K = np.concatenate([rs[r]["K"].cpu().numpy()[:rs[r]["info"].nvals] for r in range(2)])
    E = np.concatenate([rs[r]["E"].cpu().numpy()[:rs[r]["info"].n_owned_trace] for r in range(2)])
    assert np.array_equal(K, one["K"].cpu().numpy()[:one["info"].nvals])
    assert np.array_equal(E, one["E"].cpu().numpy()[:one["info"].n_owned_trace])
    ci = np.concatenate([rs[r]["col_idx"].cpu().numpy()[:rs[r]["info"].nnzb] for r in range(2)])
    assert np.array_equal(ci, one["col_idx"].cpu().numpy()[:one["info"].nnzb])


def test_singular_element_reported(cuda):
    import paper_1308_3995_b200 as hdg
    w = gen.config("C2", nr=2, nt=3)
    blk = gen.host_blocks(w)
    e_bad = 5
    A = blk["A"][blk["off_A"][e_bad]:blk["off_A"][e_bad + 1]].reshape(24, 24)
    A[:, 7] = 0.0
    r = run_gpu(w, blk=blk)
    info = r["infot"].cpu().numpy()[:w.E]
    assert info[e_bad] == 8 and (np.delete(info, e_bad) == 0).all()
    S = r["S"].cpu().numpy()
    o = w.off["S"]
    assert np.isnan(S[o[e_bad]:o[e_bad + 1]]).all()
    assert np.isfinite(np.delete(S, np.arange(o[e_bad], o[e_bad + 1]))).all()
    assert r["ctx"].first_error(r["infot"]) == (e_bad, 8)


def test_argument_errors(cuda):
    import torch
    import paper_1308_3995_b200 as hdg
    w = gen.config("C1", nr=2, nt=3)
    ctx = hdg.Context(0)
    with pytest.raises(hdg.HDGError) as ei:
        ctx.condense(*([torch.zeros(4, dtype=torch.float64, device="cuda")] * 8), torch.zeros(16, dtype=torch.uint8,
                     device="cuda"), torch.zeros(1, dtype=torch.int32, device="cuda"))
    assert ei.value.status == hdg.HDG_ERR_STATE
    ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
    x = torch.zeros(100000, dtype=torch.float64, device="cuda")
    mis = x[1:]          # 8-byte aligned, not 16
    S, g, F, inf = ctx.alloc("S"), ctx.alloc("g"), ctx.alloc("factors"), ctx.alloc("info")
    with pytest.raises(hdg.HDGError) as ei:
        ctx.condense(mis, x, x, x, x, x, S, g, F, inf)
    assert ei.value.status == hdg.HDG_ERR_ARG
    bad = w.face_elem.copy()
    bad[3] = bad[3][::-1]
    with pytest.raises(hdg.HDGError) as ei:
        ctx.plan(w.elem_face, bad, w.face_ndof, w.elem_ne)
    with pytest.raises(hdg.HDGError) as ei:
        ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne * 0 + 260)
    assert ei.value.status == hdg.HDG_ERR_UNSUPPORTED


def test_empty_slab(cuda):
    import paper_1308_3995_b200 as hdg
    w = gen.config("C1", nr=2, nt=3)
    ctx = hdg.Context(0)
    info = ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne, 0, 0)
    assert info.n_elem == 0 and info.n_owned_faces == 0 and info.nnzb == 0
    t = ctx.alloc("S")
    ctx.condense(t, t, t, t, t, t, t, t, ctx.alloc("factors"), ctx.alloc("info"))
    ctx.assemble_skeleton(t, t, ctx.alloc("K"), ctx.alloc("E"))
    ctx.backsubstitute(ctx.alloc("factors"), t, t, t, t)
    # the adjoint calls on the empty slab are no-ops too
    ctx.condense_adjoint_rhs(ctx.alloc("factors"), t, t, None, t)
    ctx.assemble_adjoint(t, t, ctx.alloc("K"), ctx.alloc("E"))
    ctx.backsubstitute_adjoint(ctx.alloc("factors"), t, t, t, t)


def test_deterministic(cuda):
    w = gen.config("C4", nr=2, nt=6)
    blk = gen.host_blocks(w)
    lam = gen.host_lambda(w)
    a, b = run_gpu(w, blk=blk, lam=lam), run_gpu(w, blk=blk, lam=lam)
    for k in ("S", "g", "K", "E", "u"):
        assert np.array_equal(a[k].cpu().numpy(), b[k].cpu().numpy()), k


def test_device_generator_bit_identical(cuda):
    import torch
    for name in ("C1", "C4"):
        w = gen.config(name, nr=2, nt=5)
        blk = gen.host_blocks(w)
        for k in ("A", "B", "C", "D", "re", "rf"):
            t = torch.empty(int(w.off[k][-1]), dtype=torch.float64, device="cuda")
            gen.device_blocks(w, k, t)
            torch.cuda.synchronize()
            assert np.array_equal(t.cpu().numpy(), blk[k]), (name, k)
    w = gen.config("C5", nr=3, nt=5)
    blk = gen.host_blocks(w)
    dne = to_dev(w.elem_ne)
    dnf = to_dev(w.elem_nf)
    for k in ("A", "C", "rf"):
        t = torch.empty(int(w.off[k][-1]), dtype=torch.float64, device="cuda")
        gen.device_blocks(w, k, t, off=to_dev(w.off[k]), dev_ne=dne, dev_nf=dnf)
        torch.cuda.synchronize()
        assert np.array_equal(t.cpu().numpy(), blk[k]), k
    lam = torch.empty(w.n_trace, dtype=torch.float64, device="cuda")
    gen.device_lambda(w, lam, to_dev(w.face_ndof), to_dev(w.face_off))
    torch.cuda.synchronize()
    assert np.array_equal(lam.cpu().numpy(), gen.host_lambda(w))
    raw = gen.device_philox_raw([[0, 0, 0, 0], [0xFFFFFFFF] * 4], [[0, 0], [0xFFFFFFFF] * 2])
    assert [hex(x) for x in raw[0]] == ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    assert [hex(x) for x in raw[1]] == ["0x408f276d", "0x41c83b0e", "0xa20bc7c6", "0x6d5451fd"]


@pytest.fixture(params=["sweep", "panel", "warp"])
def kernel(request, monkeypatch):
    """Force one condensation kernel for every bucket it supports (read by hdg_plan)."""
    monkeypatch.setenv("HDG_CONDENSE_KERNEL", request.param)
    return request.param


@pytest.mark.parametrize("name,nr,nt", [("C1", 3, 5), ("C2", 4, 9), ("C3", 5, 9), ("C4", 4, 9)])
def test_both_condense_kernels(cuda, kernel, name, nr, nt):
    """Each condensation kernel (sweep: one element per SM with register-resident [S|g]; panel: several CTAs
    per SM) is held to the same bar on every uniform config's block sizes, whichever one the plan would pick."""
    check_all(gen.config(name, nr=nr, nt=nt))


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_both_kernels_pivot_forcing(cuda, kernel, name):
    """P9 on both kernels: permuted rows force the exact (pivoting) path; a zero-ish leading entry too."""
    w = gen.config(name, nr=2, nt=4)
    blk = gen.host_blocks(w)
    rng = np.random.default_rng(7)
    for e in range(w.E):
        ne, nf = int(w.elem_ne[e]), int(w.elem_nf[e])
        A = blk["A"][blk["off_A"][e]:blk["off_A"][e + 1]].reshape(ne, ne)
        B = blk["B"][blk["off_B"][e]:blk["off_B"][e + 1]].reshape(ne, nf)
        re = blk["re"][blk["off_re"][e]:blk["off_re"][e + 1]]
        if e % 2 == 0:       # every other element pivots: fast and exact paths interleave in one CTA
            P = rng.permutation(ne)
            A[...] = A[P]
            B[...] = B[P]
            re[...] = re[P]
    check_all(w, blk=blk)


def test_sweep_hp_buckets(cuda, monkeypatch):
    """configs[4] with the sweep kernel forced: its supported (n_e, n_f) buckets next to panel-kernel buckets."""
    monkeypatch.setenv("HDG_CONDENSE_KERNEL", "sweep")
    check_all(gen.config("C5", nr=5, nt=10))


@pytest.mark.parametrize("name,nr,nt,P", [("C2", 4, 10, 2), ("C5", 4, 12, 3), ("C3", 3, 8, 4)])
def test_exchange_kernels_on_oracle_S_bitwise(cuda, name, nr, nt, P):
    """a6/a7 anchored to the oracle: the ORACLE's S and g, split into P element slabs, go through libhdg's own
    pack_kernel (inside hdg_assemble_skeleton) -> device buffer swap (the transport, done here by copies on one
    GPU) -> accumulate_kernel; the concatenated owned rows equal oracle.assemble of the whole mesh bit for bit
    (P12; left contribution first, then right)."""
    import torch
    import paper_1308_3995_b200 as hdg
    w = gen.config(name, nr=nr, nt=nt)
    ref = oracle.pipeline(w, lam=np.zeros(w.n_trace))
    c = ref["cond"]
    reb = np.array([(r * w.E) // P for r in range(P + 1)], dtype=np.int64)
    reb[1] -= 3                                   # uneven slabs
    ranks = []
    for r in range(P):
        eb, n = int(reb[r]), int(reb[r + 1] - reb[r])
        ctx = hdg.Context(0, r, P)
        info = ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne, eb, n, reb)
        S = to_dev(c["S"][c["off_S"][eb]:c["off_S"][eb + n]])
        g = to_dev(c["g"][c["off_g"][eb]:c["off_g"][eb + n]])
        K, E = ctx.alloc("K"), ctx.alloc("E")
        send = ctx.alloc("send") if info.send_doubles > 0 else None
        ctx.assemble_skeleton(S, g, K, E, send=send)
        ranks.append(dict(ctx=ctx, info=info, K=K, E=E, send=send, counts=ctx.exchange_counts()))
    for r in range(P):
        me = ranks[r]
        sc, sd, rc, rd = me["counts"]
        recv = me["ctx"].alloc("recv")
        for q in range(P):
            if q == r or rc[q] == 0:
                continue
            osc, osd, _, _ = ranks[q]["counts"]
            assert osc[r] == rc[q]
            recv[rd[q]:rd[q] + rc[q]] = ranks[q]["send"][osd[r]:osd[r] + osc[r]]
        me["ctx"].skeleton_accumulate(recv, me["K"], me["E"])
    torch.cuda.synchronize()
    K = np.concatenate([x["K"].cpu().numpy()[:x["info"].nvals] for x in ranks])
    E = np.concatenate([x["E"].cpu().numpy()[:x["info"].n_owned_trace] for x in ranks])
    assert np.array_equal(K, ref["K"])
    assert np.array_equal(E, ref["E"])


def test_nccl_context_bootstrap_single_rank(cuda):
    """The in-library NCCL bootstrap on one GPU: hdg_get_unique_id -> hdg_ctx_create with the id (a one-rank
    communicator); the context reports its communicator and the whole path still matches the oracle."""
    import paper_1308_3995_b200 as hdg
    nid = hdg.get_unique_id()
    assert len(nid) == 128
    ctx = hdg.Context(0, 0, 1, nccl_id=nid)
    assert ctx.has_comm
    w = gen.config("C2", nr=3, nt=6)
    blk = gen.host_blocks(w)
    lam = gen.host_lambda(w)
    ref = oracle.pipeline(w, blk=blk, lam=lam)
    r = run_gpu(w, blk=blk, lam=lam, ctx=ctx)
    assert np.array_equal(r["col_idx"].cpu().numpy()[:r["info"].nnzb], ref["sym"][1])
    assert rel_per_block(r["K"].cpu().numpy(), ref["K"], ref["sym"][2]) < KTOL
    ctx.close()
