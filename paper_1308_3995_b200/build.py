"""Build libhdg.so (the C-ABI library of include/hdg.h) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libhdg.so")
SOURCES = ["api.cu", "condense.cu", "condense_sweep.cu", "condense_warp.cu", "backsub.cu", "skeleton.cu", "adjoint.cu",
           "comm.cu", "condense_rows.cu", "solutions.cu",
           "skeleton_solve.cu"]
HEADERS = ["hdg_internal.cuh", "dev_common.cuh", os.path.join("..", "..", "include", "hdg.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills"]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return SO
    # the translation units compile in parallel (the sweep/panel kernels dominate: ~2 min serially)
    jobs = []
    for s in SOURCES:
        o = os.path.join(CSRC, s.replace(".cu", ".o"))
        cmd = ["nvcc", *NVCC_FLAGS, "-c", os.path.join(CSRC, s), "-o", o]
        jobs.append((s, o, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    objs, failed = [], []
    for s, o, cmd, pr in jobs:
        out, err = pr.communicate()
        if verbose or pr.returncode:
            print(" ".join(cmd))
            print(out, err)
        if pr.returncode:
            failed.append(s)
        objs.append(o)
    if failed:
        raise RuntimeError(f"nvcc failed on {failed}")
    tmp = SO + ".tmp"
    cmd = ["nvcc", "-shared", "-o", tmp, *objs, "-lcudart", "-ldl"]   # NCCL: dlopen at run time (comm.cu)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        print(r.stdout, r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    build(force=True, verbose=True)
