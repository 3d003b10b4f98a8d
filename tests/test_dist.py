"""T5: the multi-GPU path for real — torchrun, one process per GPU, NCCL over NVLink, the exchange
INSIDE libhdg (hdg_get_unique_id -> hdg_ctx_create with the id -> hdg_assemble_skeleton packs, runs one grouped
ncclSend/ncclRecv on the caller's stream and accumulates, no host sync). P12: the concatenated owned rows of K and
E at P = 2 (and 4, 8 when the GPUs exist) are bit-identical to the single-rank assembly, and match the oracle; the
distributed skeleton solve (GMRES over the slabs: NCCL halo exchange before every SpMV, all-reduced dots) returns the
same lambda on every rank, within 1e-9 of the oracle's dense solve of the whole mesh.
Skipped when fewer than 2 GPUs are visible (the round's GPU box has one; the driver's multi-GPU box runs it)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("P", [2, 4, 8])
def test_nccl_slabs_bitwise_equal_one_rank(P, tmp_path):
    if _ngpus() < P:
        pytest.skip(f"needs {P} GPUs (have {_ngpus()})")
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "res"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "dist_worker.py"),
           str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert open(str(out)).read().strip() == "ok", open(str(out)).read()
