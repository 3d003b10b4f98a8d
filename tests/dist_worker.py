"""Worker of tests/test_dist.py (launched by torchrun, one process per GPU; not collected by pytest)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main(out_path):
    import torch
    import torch.distributed as dist
    import gen
    import oracle
    import paper_1308_3995_b200 as hdg
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    msgs = []
    for name, nr, nt in (("C2", 4, 16), ("C5", 4, 16)):
        w = gen.config(name, nr=nr, nt=nt)
        blk = gen.host_blocks(w)
        reb = np.array([(r * w.E) // world for r in range(world + 1)], dtype=np.int64)
        eb, n = int(reb[rank]), int(reb[rank + 1] - reb[rank])
        ctx = hdg.nccl_context(local, rank, world)
        assert ctx.has_comm
        info = ctx.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne, eb, n, reb)
        dev = torch.device("cuda", local)
        d = {k: torch.from_numpy(blk[k][blk["off_" + k][eb]:blk["off_" + k][eb + n]].copy()).to(dev)
             for k in ("A", "B", "C", "D", "re", "rf")}
        S, g, F, inf = ctx.alloc("S"), ctx.alloc("g"), ctx.alloc("factors"), ctx.alloc("info")
        K, E = ctx.alloc("K"), ctx.alloc("E")
        stream = torch.cuda.Stream(dev)
        ctx.condense(d["A"], d["B"], d["C"], d["D"], d["re"], d["rf"], S, g, F, inf, stream=stream)
        ctx.assemble_skeleton(S, g, K, E, stream=stream)        # pack -> NCCL exchange -> accumulate, in-library
        stream.synchronize()
        Kl = K[:info.nvals].cpu()
        El = E[:info.n_owned_trace].cpu()
        parts = [None] * world
        dist.all_gather_object(parts, (Kl.numpy(), El.numpy()))
        if rank == 0:
            one = hdg.Context(local)
            i1 = one.plan(w.elem_face, w.face_elem, w.face_ndof, w.elem_ne)
            d1 = {k: torch.from_numpy(blk[k].copy()).to(dev) for k in ("A", "B", "C", "D", "re", "rf")}
            S1, g1, F1, in1 = one.alloc("S"), one.alloc("g"), one.alloc("factors"), one.alloc("info")
            K1, E1 = one.alloc("K"), one.alloc("E")
            one.condense(d1["A"], d1["B"], d1["C"], d1["D"], d1["re"], d1["rf"], S1, g1, F1, in1)
            one.assemble_skeleton(S1, g1, K1, E1)
            torch.cuda.synchronize()
            Kc = np.concatenate([p[0] for p in parts])
            Ec = np.concatenate([p[1] for p in parts])
            if not np.array_equal(Kc, K1[:i1.nvals].cpu().numpy()) or not np.array_equal(Ec, E1[:i1.n_owned_trace].cpu().numpy()):
                msgs.append(f"{name}: P={world} rows differ from one rank")
            ref = oracle.pipeline(w, blk=blk, lam=np.zeros(w.n_trace))
            bo = ref["sym"][2]
            worst = max(np.linalg.norm(Kc[bo[q]:bo[q + 1]] - ref["K"][bo[q]:bo[q + 1]]) /
                        np.linalg.norm(ref["K"][bo[q]:bo[q + 1]]) for q in range(len(bo) - 1))
            if worst > 1e-12:
                msgs.append(f"{name}: K vs oracle {worst:.2e}")
        # the distributed skeleton solve (§8(f) NEXT #3): GMRES over the slabs (halo exchange before every SpMV,
        # all-reduced dots), lambda replicated on return; the reconstruction on each slab with it
        lam = torch.zeros(w.n_trace, dtype=torch.float64, device=dev)
        it, rr = ctx.skeleton_solve(K, E, lam, rtol=1e-12, maxit=3000, restart=60, stream=stream)
        stream.synchronize()
        if rr > 1e-11:
            msgs.append(f"{name}: rank {rank} distributed solve relres {rr:.2e} after {it}")
        lams = [None] * world
        dist.all_gather_object(lams, lam.cpu().numpy())
        if rank == 0:
            ref_lam = oracle.pipeline(w, blk=blk)["lam"]            # the O5 dense solve of the whole mesh
            for q in range(world):
                err = np.linalg.norm(lams[q] - ref_lam) / np.linalg.norm(ref_lam)
                if err > 1e-9:
                    msgs.append(f"{name}: P={world} lambda on rank {q} vs the dense oracle {err:.2e}")
        ctx.close()
        dist.barrier()
    if rank == 0:
        open(out_path, "w").write("ok" if not msgs else "; ".join(msgs))
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
