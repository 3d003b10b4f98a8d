"""gen — seeded synthetic inputs shared by the oracle tests and the CUDA path.

Holds none of the method's arithmetic (no factorisation, Schur complement, assembly or back-substitution).
It builds the BASELINE.json workloads:

* the periodic annulus triangulation (stand-in for the paper's NACA0012 meshes, which are not in the
  container; connectivity only, §3.1),
* the degree map and hp sizes n_e = m_e n(p), n(p) = (p+1)(p+2)/2, trace size
  m_t (p_f+1) with p_f = max(p_K-, p_K+),
* element blocks A, B, C, D, r_e, r_f and a trace vector lambda from Philox4x32-10 (gen/philox_normal.h),
  on the host (gen_host.c) or directly in device memory (gen_device.cu), bit-identical either way.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HOST_SO = os.path.join(_HERE, "libhdggen.so")
_DEV_SO = os.path.join(_HERE, "libhdggen_dev.so")

KIND_A, KIND_B, KIND_C, KIND_D, KIND_RE, KIND_RF = range(6)
TAG_LAMBDA = 8
SEED_BASE = 0x13083995


def build(verbose: bool = False, device: bool = True) -> None:
    """Compile the host generator (gcc, no FMA contraction) and the device generator (nvcc --fmad=false)."""
    src = os.path.join(_HERE, "gen_host.c")
    if not os.path.exists(_HOST_SO) or os.path.getmtime(_HOST_SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "philox_normal.h"))):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
               "-o", _HOST_SO, src, "-lm"]
        subprocess.run(cmd, check=True, capture_output=not verbose)
    if device:
        dsrc = os.path.join(_HERE, "gen_device.cu")
        if not os.path.exists(_DEV_SO) or os.path.getmtime(_DEV_SO) < max(
                os.path.getmtime(dsrc), os.path.getmtime(os.path.join(_HERE, "philox_normal.h"))):
            cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false",
                   "-Xcompiler", "-fPIC", "-shared", "-o", _DEV_SO, dsrc]
            subprocess.run(cmd, check=True, capture_output=not verbose)


_host = None
_dev = None


def _lib():
    global _host
    if _host is None:
        build(device=False)
        lib = ctypes.CDLL(_HOST_SO)
        P = ctypes.c_void_p
        lib.gen_annulus.restype = ctypes.c_int64
        lib.gen_annulus.argtypes = [ctypes.c_int32, ctypes.c_int32, P, P]
        lib.gen_degrees.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, P]
        lib.gen_blocks.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, P, P] + [P] * 12
        lib.gen_lambda.argtypes = [ctypes.c_uint64, ctypes.c_int64, P, P, P]
        lib.gen_philox_raw.argtypes = [P, P, P]
        lib.gen_normals.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int64, P]
        lib.gen_ln_det.restype = ctypes.c_double
        lib.gen_ln_det.argtypes = [ctypes.c_double]
        lib.gen_sincos_2pi_det.argtypes = [ctypes.c_double, P, P]
        _host = lib
    return _host


def _devlib():
    global _dev
    if _dev is None:
        build(device=True)
        lib = ctypes.CDLL(_DEV_SO)
        P = ctypes.c_void_p
        lib.gen_dev_blocks.restype = ctypes.c_int
        lib.gen_dev_blocks.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, P, P, P,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int64, P, P]
        lib.gen_dev_lambda.restype = ctypes.c_int
        lib.gen_dev_lambda.argtypes = [ctypes.c_uint64, ctypes.c_int64, P, P, P, P]
        lib.gen_dev_philox_raw.restype = ctypes.c_int
        lib.gen_dev_philox_raw.argtypes = [P, P, P, ctypes.c_int, P]
        _dev = lib
    return _dev


def _ptr(a) -> ctypes.c_void_p:
    if a is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(a.ctypes.data)


# ----------------------------------------------------------------------------------------------------------
# raw generator access (pins)

def philox_raw(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    _lib().gen_philox_raw(_ptr(c), _ptr(k), _ptr(out))
    return out


def normals(seed: int, id_: int, tag: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _lib().gen_normals(seed, id_, tag, n, _ptr(out))
    return out


def det_ln(x: float) -> float:
    return _lib().gen_ln_det(x)


def det_sincos_2pi(u: float):
    s, c = ctypes.c_double(), ctypes.c_double()
    _lib().gen_sincos_2pi_det(u, ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


# ----------------------------------------------------------------------------------------------------------
# mesh and degree map

def annulus(nr: int, nt: int):
    """Connectivity of the periodic annulus. Returns (elem_face[E,3], face_elem[F,2])."""
    E = 2 * nr * nt
    F = (3 * nr + 1) * nt
    ef = np.empty((E, 3), dtype=np.int32)
    fe = np.empty((F, 2), dtype=np.int32)
    got = _lib().gen_annulus(nr, nt, _ptr(ef), _ptr(fe))
    assert got == F, (got, F)
    return ef, fe


def degrees(seed: int, E: int, p_fixed: int) -> np.ndarray:
    p = np.empty(E, dtype=np.int32)
    _lib().gen_degrees(seed, E, p_fixed, _ptr(p))
    return p


def n_modes(p):
    return (np.asarray(p) + 1) * (np.asarray(p) + 2) // 2


@dataclass
class Workload:
    """One synthetic workload: mesh, degree map, per-element sizes and dense-packed block offsets."""
    name: str
    seed: int
    nr: int
    nt: int
    m_elem: int            # element unknowns per mode: 4 (Euler, W only) or 12 (NS mixed: W + 2D gradient Q)
    m_trace: int           # trace unknowns per edge mode (4)
    p_fixed: int           # >0 uniform degree; 0 = hp draw
    boundary: str = "all"  # "all": boundary faces carry one-sided trace rows; "paper": Gamma_h only
    elem_face: np.ndarray = field(default=None, repr=False)
    face_elem: np.ndarray = field(default=None, repr=False)
    p: np.ndarray = field(default=None, repr=False)
    face_p: np.ndarray = field(default=None, repr=False)
    face_ndof: np.ndarray = field(default=None, repr=False)
    elem_ne: np.ndarray = field(default=None, repr=False)
    elem_nf: np.ndarray = field(default=None, repr=False)
    face_off: np.ndarray = field(default=None, repr=False)
    off: dict = field(default=None, repr=False)   # name -> int64[E+1] offsets in doubles (dense packing)

    @property
    def E(self) -> int:
        return int(self.elem_face.shape[0])

    @property
    def F(self) -> int:
        return int(self.face_elem.shape[0])

    @property
    def n_trace(self) -> int:
        return int(self.face_off[-1])

    @property
    def uniform(self) -> bool:
        return bool((self.elem_ne == self.elem_ne[0]).all() and (self.elem_nf == self.elem_nf[0]).all())

    def sizes(self, name: str) -> np.ndarray:
        a, f = self.elem_ne.astype(np.int64), self.elem_nf.astype(np.int64)
        return {"A": a * a, "B": a * f, "C": f * a, "D": f * f, "re": a, "rf": f, "S": f * f, "g": f,
                "u": a}[name]


ARRAYS = ("A", "B", "C", "D", "re", "rf", "S", "g", "u")


def make_workload(name: str, nr: int, nt: int, m_elem: int, p_fixed: int, seed: int, m_trace: int = 4,
                  boundary: str = "all") -> Workload:
    ef, fe = annulus(nr, nt)
    E = ef.shape[0]
    p = degrees(seed, E, p_fixed)
    if boundary == "paper":
        # Gamma_h excludes boundary edges; lambda_h is not defined there.
        interior = fe[:, 1] >= 0
        new_id = np.full(fe.shape[0], -1, dtype=np.int64)
        new_id[interior] = np.arange(int(interior.sum()))
        ef = np.where(ef >= 0, new_id[ef], -1).astype(np.int32)
        fe = np.ascontiguousarray(fe[interior])
    elif boundary != "all":
        raise ValueError(boundary)
    pl = p[fe[:, 0]]
    pr = np.where(fe[:, 1] >= 0, p[np.maximum(fe[:, 1], 0)], pl)
    face_p = np.maximum(pl, pr).astype(np.int32)          # p_e = max(p_K-, p_K+)
    face_ndof = (m_trace * (face_p + 1)).astype(np.int32)
    nf = np.where(ef >= 0, face_ndof[np.maximum(ef, 0)], 0).sum(axis=1).astype(np.int32)
    ne = (m_elem * n_modes(p)).astype(np.int32)
    face_off = np.zeros(fe.shape[0] + 1, dtype=np.int64)
    np.cumsum(face_ndof, out=face_off[1:])
    w = Workload(name=name, seed=seed, nr=nr, nt=nt, m_elem=m_elem, m_trace=m_trace, p_fixed=p_fixed,
                 boundary=boundary, elem_face=ef, face_elem=fe, p=p, face_p=face_p, face_ndof=face_ndof,
                 elem_ne=ne, elem_nf=nf, face_off=face_off)
    w.off = {}
    for a in ARRAYS:
        o = np.zeros(E + 1, dtype=np.int64)
        np.cumsum(w.sizes(a), out=o[1:])
        w.off[a] = o
    return w


# BASELINE.json configs[0..4]
CONFIGS = {
    "C1": dict(nr=16, nt=32, m_elem=4, p_fixed=1),
    "C2": dict(nr=64, nt=128, m_elem=4, p_fixed=2),
    "C3": dict(nr=256, nt=512, m_elem=4, p_fixed=4),
    "C4": dict(nr=128, nt=512, m_elem=12, p_fixed=3),
    "C5": dict(nr=512, nt=1024, m_elem=12, p_fixed=0),
}


def config(name: str, boundary: str = "all", nr: int | None = None, nt: int | None = None) -> Workload:
    """BASELINE.json config by name; nr/nt override the mesh size (same block sizes, smaller meshes)."""
    c = dict(CONFIGS[name])
    if nr is not None:
        c["nr"] = nr
    if nt is not None:
        c["nt"] = nt
    idx = int(name[1])
    return make_workload(name, seed=SEED_BASE + idx, boundary=boundary, **c)


# ----------------------------------------------------------------------------------------------------------
# blocks

def host_blocks(w: Workload, e0: int = 0, n: int | None = None, which=("A", "B", "C", "D", "re", "rf")) -> dict:
    """Blocks of elements [e0, e0+n) as dense-packed float64 arrays with local offsets (key 'off_*')."""
    if n is None:
        n = w.E - e0
    ne = np.ascontiguousarray(w.elem_ne[e0:e0 + n])
    nf = np.ascontiguousarray(w.elem_nf[e0:e0 + n])
    out = {}
    offs = {}
    for a in ("A", "B", "C", "D", "re", "rf"):
        o = w.off[a][e0:e0 + n + 1] - w.off[a][e0]
        offs[a] = np.ascontiguousarray(o)
        out["off_" + a] = offs[a]
        out[a] = np.empty(int(o[-1]), dtype=np.float64) if a in which else None
    _lib().gen_blocks(w.seed, e0, n, _ptr(ne), _ptr(nf),
                      *[_ptr(offs[a]) for a in ("A", "B", "C", "D", "re", "rf")],
                      *[_ptr(out[a]) for a in ("A", "B", "C", "D", "re", "rf")])
    return out


def host_lambda(w: Workload, seed: int | None = None) -> np.ndarray:
    lam = np.empty(w.n_trace, dtype=np.float64)
    _lib().gen_lambda(w.seed if seed is None else seed, w.F, _ptr(w.face_ndof), _ptr(w.face_off), _ptr(lam))
    return lam


_KIND = {"A": KIND_A, "B": KIND_B, "C": KIND_C, "D": KIND_D, "re": KIND_RE, "rf": KIND_RF}


def device_blocks(w: Workload, name: str, out, e0: int = 0, n: int | None = None, off=None, stream=None,
                  dev_ne=None, dev_nf=None):
    """Fill the torch float64 CUDA tensor `out` with block `name` of elements [e0, e0+n).

    Uniform workloads use a constant stride; ragged ones need device int32 ne/nf and int64 offsets `off`
    (local to e0). Bit-identical to host_blocks."""
    import torch
    if n is None:
        n = w.E - e0
    s = torch.cuda.current_stream().cuda_stream if stream is None else stream
    if w.uniform and off is None:
        a, f = int(w.elem_ne[0]), int(w.elem_nf[0])
        stride = int(w.sizes(name)[0])
        rc = _devlib().gen_dev_blocks(w.seed, e0, n, _KIND[name], None, None, None, a, f, stride,
                                      ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s))
    else:
        rc = _devlib().gen_dev_blocks(w.seed, e0, n, _KIND[name], ctypes.c_void_p(dev_ne.data_ptr()),
                                      ctypes.c_void_p(dev_nf.data_ptr()), ctypes.c_void_p(off.data_ptr()),
                                      0, 0, 0, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s))
    if rc != 0:
        raise RuntimeError(f"gen_dev_blocks failed: cudaError {rc}")


def device_lambda(w: Workload, out, dev_face_ndof, dev_face_off, seed: int | None = None):
    import torch
    s = torch.cuda.current_stream().cuda_stream
    rc = _devlib().gen_dev_lambda(w.seed if seed is None else seed, w.F, ctypes.c_void_p(dev_face_ndof.data_ptr()),
                                  ctypes.c_void_p(dev_face_off.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                  ctypes.c_void_p(s))
    if rc != 0:
        raise RuntimeError(f"gen_dev_lambda failed: cudaError {rc}")


def device_philox_raw(ctr, key):
    import torch
    c = torch.as_tensor(np.ascontiguousarray(ctr, dtype=np.uint32).view(np.int32)).cuda()
    k = torch.as_tensor(np.ascontiguousarray(key, dtype=np.uint32).view(np.int32)).cuda()
    n = c.numel() // 4
    o = torch.empty(4 * n, dtype=torch.int32, device="cuda")
    rc = _devlib().gen_dev_philox_raw(ctypes.c_void_p(c.data_ptr()), ctypes.c_void_p(k.data_ptr()),
                                      ctypes.c_void_p(o.data_ptr()), n,
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    return o.cpu().numpy().view(np.uint32).reshape(n, 4)


# ------------------------------------------------------------------------------------------------------------
# Pseudo-time relaxation inputs (§8(f) NEXT #4). These are INPUTS of the re-condensation (like
# A_e), not the method's arithmetic: a CFL number per Newton step from the paper's ramp, and per element a
# seeded stand-in for the spectral-radius estimate (lambda_c + 4 lambda_v) of the local time step
# dt_K = CFL |K| / (lambda_c + 4 lambda_v).
def cfl_ramp(n: int, n0: int = 10, c0: float = 10.0) -> float:
    """CFL^n for n <= n0: c0 (3 (n/n0)^2 - 2 (n/n0)^3) (PAPER.md eq. cfl, the ramping phase)."""
    x = min(max(n / n0, 0.0), 1.0)
    return c0 * (3.0 * x * x - 2.0 * x * x * x)


def pseudo_time_shift(w: Workload, cfl: float, e0: int = 0, n: int | None = None) -> np.ndarray:
    """Per-element diagonal shift packed like r_e: |K| / dt_K = (lambda_c + 4 lambda_v)_K / CFL on the element's
    w unknowns (an orthonormal modal basis: M_e = |K| I), 0 on the gradient unknowns q. Element unknowns are
    [Q; W] basis-major (DESIGN R4): for NS mixed (m_elem = 12) W is the last 4 n(p) unknowns, for Euler all.
    The spectral-radius stand-in is 1 + |z_K| with z_K ~ N(0, 1) from a seeded numpy generator (keyed by the
    workload seed and the element id, so slabs agree)."""
    if n is None:
        n = w.E - e0
    lam = np.empty(n)
    for k in range(n):
        rng = np.random.default_rng([w.seed, 9, e0 + k])
        lam[k] = 1.0 + abs(rng.standard_normal())
    out = np.zeros(int(w.off["re"][e0 + n] - w.off["re"][e0]))
    o = 0
    for k in range(n):
        ne = int(w.elem_ne[e0 + k])
        nw = 4 * (ne // w.m_elem) if w.m_elem != 4 else ne
        out[o + ne - nw:o + ne] = lam[k] / cfl
        o += ne
    return out
