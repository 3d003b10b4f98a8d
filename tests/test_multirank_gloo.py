"""The N > 1 path on CPU (no GPU): world-size-2 `torch.distributed` over gloo, 127.0.0.1.

Each rank owns an element slab. Its shared-face contributions follow libhdg's exchange layout
(hdg_exchange_layout — the host code hdg_plan uses, callable without a device) and travel through the product's
transport (paper_1308_3995_b200.exchange_buffers: torch.distributed point-to-point ops; NCCL for CUDA tensors in
bench.py, gloo here). Packing and the ordered accumulation, which run in libhdg's CUDA kernels on the GPU
(pack_kernel / accumulate_kernel, covered by test_parity_gpu.py::test_two_rank_slabs_bitwise_equal_one_rank), are
restated here in numpy from the layout's documented packing (include/hdg.h). The concatenated owned rows must equal
the single-rank oracle assembly bit for bit (P12; left contribution first, then right).
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slot_offset(w, e, f):
    o = 0
    for c in w.elem_face[e]:
        if c == f:
            return o
        if c >= 0:
            o += int(w.face_ndof[c])
    raise AssertionError((e, f))


def _rank_main(rank, world, port, name, nr, nt, boundary, out_q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import gen
    import oracle
    import paper_1308_3995_b200 as hdg
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        w = gen.config(name, nr=nr, nt=nt, boundary=boundary)
        rb = np.array([(r * w.E) // world for r in range(world + 1)], dtype=np.int64)
        eb, n = int(rb[rank]), int(rb[rank + 1] - rb[rank])
        blk = gen.host_blocks(w, eb, n)
        c = oracle.condense(w.elem_ne[eb:eb + n], w.elem_nf[eb:eb + n], blk)
        lay = hdg.exchange_layout(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne, rb, rank)
        # pack (the documented layout): [g_l[slot f] | S_l[slot f rows, all columns]]
        send = torch.zeros(max(1, int(lay["send_counts"].sum())), dtype=torch.float64)
        for f, l, o in lay["send_items"]:
            e = eb + int(l)
            na, nfl = int(w.face_ndof[f]), int(w.elem_nf[e])
            so = _slot_offset(w, e, int(f))
            g = c["g"][c["off_g"][l]:c["off_g"][l + 1]]
            S = c["S"][c["off_S"][l]:c["off_S"][l + 1]].reshape(nfl, nfl)
            send[o:o + na] = torch.from_numpy(g[so:so + na].copy())
            send[o + na:o + na + na * nfl] = torch.from_numpy(S[so:so + na].reshape(-1).copy())
        recv = torch.zeros(max(1, int(lay["recv_counts"].sum())), dtype=torch.float64)
        hdg.exchange_buffers(send, recv, lay["send_counts"], lay["send_displs"], lay["recv_counts"],
                             lay["recv_displs"], rank, world)
        # owned rows = faces whose left element is local; local (left) contributions first
        owned = np.nonzero((w.face_elem[:, 0] >= eb) & (w.face_elem[:, 0] < eb + n))[0]
        f0, f1 = int(owned.min()), int(owned.max()) + 1
        assert f1 - f0 == len(owned)            # a contiguous id range (S16)
        sym = oracle.symbolic(w.elem_face, w.face_elem, w.face_ndof, f0, f1)
        K, E = oracle.assemble(w.elem_face, w.face_ndof, w.face_off, w.elem_nf[eb:eb + n], c["S"], c["off_S"], c["g"],
                               c["off_g"], sym, f0, f1, eb, n)
        rp, ci, bo = sym
        rv = recv.numpy()
        for f, e, o in lay["recv_items"]:
            f, e, o = int(f), int(e), int(o)
            na, nfe = int(w.face_ndof[f]), int(w.elem_nf[e])
            tr = int(w.face_off[f] - w.face_off[f0])
            E[tr:tr + na] = E[tr:tr + na] + rv[o:o + na]
            strip = rv[o + na:o + na + na * nfe].reshape(na, nfe)
            soff = 0
            for cf in w.elem_face[e]:
                if cf < 0:
                    continue
                nb = int(w.face_ndof[cf])
                q = [j for j in range(rp[f - f0], rp[f - f0 + 1]) if ci[j] == cf][0]
                blkv = K[bo[q]:bo[q] + na * nb].reshape(na, nb)
                blkv[...] = blkv + strip[:, soff:soff + nb]
                soff += nb
        out_q.put((rank, f0, f1, K, E, int(lay["send_counts"].sum()), int(lay["recv_counts"].sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,nr,nt,boundary", [("C2", 4, 10, "all"), ("C5", 3, 8, "all"), ("C3", 2, 6, "paper")])
def test_two_rank_gloo_assembly_bitwise(name, nr, nt, boundary):
    import torch.multiprocessing as mp
    sys.path.insert(0, ROOT)
    import gen
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, name, nr, nt, boundary, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = gen.config(name, nr=nr, nt=nt, boundary=boundary)
    ref = oracle.pipeline(w, lam=np.zeros(w.n_trace))
    K_all = np.concatenate([r[3] for r in res])
    E_all = np.concatenate([r[4] for r in res])
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == w.F
    assert np.array_equal(K_all, ref["K"])
    assert np.array_equal(E_all, ref["E"])
    assert res[0][6] > 0 and res[1][5] > 0      # the exchange carried shared-face rows both ways it had to
