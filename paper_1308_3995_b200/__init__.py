"""paper_1308_3995_b200 — B200-native static condensation for hybridized DG (arXiv 1308.3995, §3.4).

Thin Python binding of libhdg.so (the C ABI in include/hdg.h): argument marshalling only. Every step of the hot
path — condensation (LU with partial pivoting, local solves, Schur complement), skeleton assembly (block-CSR,
left-then-right sums), the shared-face exchange pack/accumulate and the back-substitution — runs in the
library's sm_100a CUDA kernels. PyTorch supplies device memory, streams and torch.distributed (plumbing only).

There is no CPU fallback: if libhdg.so is missing or no sm_100 device is present, every call raises.

Names follow the paper: K, E (Eq. hybridsystem), lambda (the trace unknowns dLambda), and the
per-element blocks A_e, B_e, C_e, D_e, r_e, r_f, S_e, g_e, u_e of SURVEY.md §0.1.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhdg.so")

(HDG_OK, HDG_ERR_ARG, HDG_ERR_SINGULAR, HDG_ERR_CUDA, HDG_ERR_NOMEM, HDG_ERR_STATE, HDG_ERR_UNSUPPORTED,
 HDG_ERR_NCCL) = range(8)


class HDGError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libhdg status {status}: {msg}")
        self.status = status


class _Mesh(ctypes.Structure):
    _fields_ = [("n_elem_global", ctypes.c_int64), ("n_face", ctypes.c_int64), ("elem_begin", ctypes.c_int64),
                ("n_elem", ctypes.c_int64), ("elem_face", ctypes.c_void_p), ("face_elem", ctypes.c_void_p),
                ("face_ndof", ctypes.c_void_p), ("elem_ndof", ctypes.c_void_p),
                ("rank_elem_begin", ctypes.c_void_p)]


class _PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "n_elem", "len_A", "len_B", "len_C", "len_D", "len_re", "len_rf", "len_S", "len_g", "len_u",
        "factor_bytes", "owned_face_begin", "n_owned_faces", "nnzb", "nvals", "owned_trace_begin",
        "n_owned_trace", "n_trace")] + [("n_buckets", ctypes.c_int32), ("max_ne", ctypes.c_int32),
                                        ("max_nf", ctypes.c_int32), ("send_doubles", ctypes.c_int64),
                                        ("recv_doubles", ctypes.c_int64), ("len_X", ctypes.c_int64)]


_lib = None


def lib():
    """Load libhdg.so. Raises if the extension has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libhdg.so not built ({LIB_PATH}); run __graft_entry__.build() or "
                              f"python paper_1308_3995_b200/build.py")
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.hdg_version.restype = ctypes.c_char_p
        L.hdg_status_string.restype = ctypes.c_char_p
        L.hdg_status_string.argtypes = [I32]
        L.hdg_ctx_create.restype = I32
        L.hdg_ctx_create.argtypes = [ctypes.POINTER(P), I32, I32, I32, P]
        L.hdg_get_unique_id.restype = I32
        L.hdg_get_unique_id.argtypes = [P]
        L.hdg_ctx_has_comm.restype = I32
        L.hdg_ctx_has_comm.argtypes = [P]
        L.hdg_ctx_destroy.argtypes = [P]
        L.hdg_last_error.restype = ctypes.c_char_p
        L.hdg_last_error.argtypes = [P]
        L.hdg_plan.restype = I32
        L.hdg_plan.argtypes = [P, ctypes.POINTER(_Mesh), ctypes.POINTER(_PlanInfo), P]
        L.hdg_condense.restype = I32
        L.hdg_condense.argtypes = [P] + [P] * 10 + [P]
        L.hdg_condense_shifted.restype = I32
        L.hdg_condense_shifted.argtypes = [P] + [P] * 11 + [P]
        L.hdg_condense_assemble.restype = I32
        L.hdg_condense_assemble.argtypes = [P] + [P] * 10 + [P]
        L.hdg_skeleton_structure.restype = I32
        L.hdg_skeleton_structure.argtypes = [P, P, P, P, P]
        L.hdg_condense_saved.restype = I32
        L.hdg_condense_saved.argtypes = [P] + [P] * 11 + [P]
        L.hdg_save_solutions.restype = I32
        L.hdg_save_solutions.argtypes = [P] + [P] * 4 + [P]
        L.hdg_backsubstitute_saved.restype = I32
        L.hdg_backsubstitute_saved.argtypes = [P] + [P] * 3 + [P]
        L.hdg_skeleton_spmv.restype = I32
        L.hdg_skeleton_spmv.argtypes = [P, P, P, P, P]
        L.hdg_skeleton_solve.restype = I32
        L.hdg_skeleton_solve.argtypes = [P, P, P, P, ctypes.c_double, I32, I32, ctypes.POINTER(I32),
                                         ctypes.POINTER(ctypes.c_double), P]
        L.hdg_nnz_counts.restype = I32
        L.hdg_nnz_counts.argtypes = [ctypes.POINTER(_Mesh), P, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.hdg_assemble_skeleton.restype = I32
        L.hdg_assemble_skeleton.argtypes = [P] + [P] * 8 + [P]
        L.hdg_exchange_counts.restype = I32
        L.hdg_exchange_counts.argtypes = [P, P, P, P, P]
        L.hdg_skeleton_accumulate.restype = I32
        L.hdg_skeleton_accumulate.argtypes = [P, P, P, P, P]
        L.hdg_backsubstitute.restype = I32
        L.hdg_backsubstitute.argtypes = [P] + [P] * 5 + [P]
        L.hdg_condense_adjoint_rhs.restype = I32
        L.hdg_condense_adjoint_rhs.argtypes = [P] + [P] * 5 + [P]
        L.hdg_assemble_adjoint.restype = I32
        L.hdg_assemble_adjoint.argtypes = [P] + [P] * 5 + [P]
        L.hdg_backsubstitute_adjoint.restype = I32
        L.hdg_backsubstitute_adjoint.argtypes = [P] + [P] * 5 + [P]
        L.hdg_first_error.restype = I32
        L.hdg_first_error.argtypes = [P, P, ctypes.POINTER(I64), ctypes.POINTER(ctypes.c_int32), P]
        L.hdg_launch_count.restype = I64
        L.hdg_launch_count.argtypes = [P]
        L.hdg_debug_set_trace.restype = I32
        L.hdg_debug_set_trace.argtypes = [P, P]
        L.hdg_max_elem_ndof.restype = I32
        L.hdg_max_face_ndof.restype = I32
        L.hdg_exchange_layout.restype = I32
        L.hdg_exchange_layout.argtypes = [ctypes.POINTER(_Mesh), I32, I32] + [P] * 8
        _lib = L
    return _lib


EXPORTED = ("hdg_version", "hdg_max_elem_ndof", "hdg_max_face_ndof", "hdg_status_string", "hdg_get_unique_id",
            "hdg_ctx_create", "hdg_ctx_has_comm",
            "hdg_ctx_destroy", "hdg_last_error", "hdg_plan", "hdg_condense", "hdg_assemble_skeleton",
            "hdg_exchange_counts", "hdg_skeleton_accumulate", "hdg_backsubstitute", "hdg_first_error",
            "hdg_launch_count", "hdg_debug_set_trace", "hdg_exchange_layout", "hdg_condense_adjoint_rhs",
            "hdg_assemble_adjoint", "hdg_backsubstitute_adjoint", "hdg_condense_shifted", "hdg_nnz_counts",
            "hdg_save_solutions", "hdg_backsubstitute_saved", "hdg_skeleton_spmv", "hdg_skeleton_solve",
            "hdg_condense_saved", "hdg_condense_assemble", "hdg_skeleton_structure")


def _ptr(t):
    if t is None:
        return ctypes.c_void_p(0)
    import torch
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if not t.is_cuda:
            raise ValueError("tensor must live on the CUDA device (libhdg takes device pointers)")
        return ctypes.c_void_p(t.data_ptr())
    raise TypeError(type(t))


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _f64(*ts):
    import torch
    for t in ts:
        if t is not None and t.dtype != torch.float64:
            raise TypeError("fp64 tensors required")


@dataclass
class PlanInfo:
    n_elem: int
    len_A: int
    len_B: int
    len_C: int
    len_D: int
    len_re: int
    len_rf: int
    len_S: int
    len_g: int
    len_u: int
    factor_bytes: int
    owned_face_begin: int
    n_owned_faces: int
    nnzb: int
    nvals: int
    owned_trace_begin: int
    n_owned_trace: int
    n_trace: int
    n_buckets: int
    max_ne: int
    max_nf: int
    send_doubles: int
    recv_doubles: int
    len_X: int


def get_unique_id() -> bytes:
    """hdg_get_unique_id: a fresh 128-byte NCCL id (call on one rank, distribute to the others)."""
    buf = ctypes.create_string_buffer(128)
    st = lib().hdg_get_unique_id(buf)
    if st != HDG_OK:
        raise HDGError(st, "hdg_get_unique_id: NCCL unavailable")
    return buf.raw


class Context:
    """One libhdg context (device, rank of nranks). Mirrors include/hdg.h call for call.
    nccl_id (128 bytes from get_unique_id, the same on every rank): the context creates its own NCCL communicator
    and hdg_assemble_skeleton / hdg_assemble_adjoint perform the shared-face exchange inside the call."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None):
        self._L = lib()
        h = ctypes.c_void_p()
        idbuf = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be 128 bytes")
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        st = self._L.hdg_ctx_create(ctypes.byref(h), device, rank, nranks, idbuf)
        if st != HDG_OK:
            raise HDGError(st, f"hdg_ctx_create(device={device}): {self._L.hdg_status_string(st).decode()}")
        self._h = h
        self.device, self.rank, self.nranks = device, rank, nranks
        self.has_comm = bool(self._L.hdg_ctx_has_comm(h))
        self.info: PlanInfo | None = None
        self._keep = None

    def close(self):
        if getattr(self, "_h", None):
            self._L.hdg_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int, what: str):
        if st != HDG_OK:
            raise HDGError(st, f"{what}: {self._L.hdg_last_error(self._h).decode()}")

    # -- a0 ------------------------------------------------------------------------------------------------------
    def plan(self, elem_face, face_elem, face_ndof, elem_ndof, elem_begin: int = 0, n_elem: int | None = None,
             rank_elem_begin=None, stream=None) -> PlanInfo:
        ef = np.ascontiguousarray(elem_face, dtype=np.int32)
        fe = np.ascontiguousarray(face_elem, dtype=np.int32)
        fn = np.ascontiguousarray(face_ndof, dtype=np.int32)
        en = np.ascontiguousarray(elem_ndof, dtype=np.int32)
        E = ef.shape[0]
        if n_elem is None:
            n_elem = E - elem_begin
        rb = None if rank_elem_begin is None else np.ascontiguousarray(rank_elem_begin, dtype=np.int64)
        m = _Mesh(E, fe.shape[0], elem_begin, n_elem, ef.ctypes.data, fe.ctypes.data, fn.ctypes.data, en.ctypes.data,
                  rb.ctypes.data if rb is not None else None)
        pi = _PlanInfo()
        self._check(self._L.hdg_plan(self._h, ctypes.byref(m), ctypes.byref(pi), _stream(stream)), "hdg_plan")
        self.info = PlanInfo(**{k: getattr(pi, k) for k, _ in _PlanInfo._fields_})
        return self.info

    def alloc(self, what: str):
        """Allocate a correctly sized device output: 'S', 'g', 'u', 'factors', 'info', 'K', 'E', 'row_ptr',
        'col_idx', 'blk_off', 'send', 'recv'."""
        import torch
        i, dev = self.info, torch.device("cuda", self.device)
        f64 = dict(dtype=torch.float64, device=dev)
        sizes = {"S": i.len_S, "g": i.len_g, "u": i.len_u, "K": i.nvals, "E": i.n_owned_trace,
                 "send": i.send_doubles, "recv": i.recv_doubles, "X": i.len_X}
        if what in sizes:
            return torch.empty(max(sizes[what], 1), **f64)
        if what == "factors":
            return torch.empty(max(i.factor_bytes, 16), dtype=torch.uint8, device=dev)
        if what == "info":
            return torch.empty(max(i.n_elem, 1), dtype=torch.int32, device=dev)
        if what == "row_ptr":
            return torch.empty(i.n_owned_faces + 1, dtype=torch.int32, device=dev)
        if what == "col_idx":
            return torch.empty(max(i.nnzb, 1), dtype=torch.int32, device=dev)
        if what == "blk_off":
            return torch.empty(i.nnzb + 1, dtype=torch.int64, device=dev)
        raise KeyError(what)

    # -- a1-a5 ---------------------------------------------------------------------------------------------------
    def condense(self, A, B, C, D, r_e, r_f, S, g, factors, info, stream=None):
        _f64(A, B, C, D, r_e, r_f, S, g)
        self._check(self._L.hdg_condense(self._h, *map(_ptr, (A, B, C, D, r_e, r_f, S, g, factors, info)),
                                         _stream(stream)), "hdg_condense")

    def condense_shifted(self, A, B, C, D, r_e, r_f, shift, S, g, factors, info, stream=None):
        """Re-condensation of A_e + diag(shift_e) (shift packed like r_e): the pseudo-time term M_e / dt_K of
        PAPER.md:303-313 with an orthonormal basis (§8(f) NEXT #4)."""
        _f64(A, B, C, D, r_e, r_f, shift, S, g)
        self._check(self._L.hdg_condense_shifted(self._h, *map(_ptr, (A, B, C, D, r_e, r_f, shift, S, g, factors,
                                                                      info)), _stream(stream)), "hdg_condense_shifted")

    # -- a6 / a7 ---------------------------------------------------------------------------------------------------
    def assemble_skeleton(self, S, g, K, E, row_ptr=None, col_idx=None, blk_off=None, send=None, stream=None):
        _f64(S, g, K, E, send)
        self._check(self._L.hdg_assemble_skeleton(self._h, *map(_ptr, (S, g, row_ptr, col_idx, blk_off, K, E, send)),
                                                  _stream(stream)), "hdg_assemble_skeleton")

    def exchange_counts(self):
        n = self.nranks
        arrs = [np.zeros(n, dtype=np.int64) for _ in range(4)]
        self._check(self._L.hdg_exchange_counts(self._h, *[ctypes.c_void_p(a.ctypes.data) for a in arrs]),
                    "hdg_exchange_counts")
        return tuple(arrs)

    def skeleton_accumulate(self, recv, K, E, stream=None):
        _f64(recv, K, E)
        self._check(self._L.hdg_skeleton_accumulate(self._h, _ptr(recv), _ptr(K), _ptr(E), _stream(stream)),
                    "hdg_skeleton_accumulate")

    # -- a8 ----------------------------------------------------------------------------------------------------------
    def backsubstitute(self, factors, B, r_e, lam, u, stream=None):
        _f64(B, r_e, lam, u)
        self._check(self._L.hdg_backsubstitute(self._h, *map(_ptr, (factors, B, r_e, lam, u)), _stream(stream)),
                    "hdg_backsubstitute")

    # ---- the skeleton solve: SURVEY.md §8(f) NEXT #3, PAPER.md:357-362 -----------------------------------------------
    def skeleton_spmv(self, K, x, y, stream=None):
        """y = K x over the owned rows (x: global trace vector)."""
        _f64(K, x, y)
        self._check(self._L.hdg_skeleton_spmv(self._h, _ptr(K), _ptr(x), _ptr(y), _stream(stream)),
                    "hdg_skeleton_spmv")

    def skeleton_solve(self, K, E, lam, rtol=1e-10, maxit=500, restart=40, stream=None):
        """K lam = E by block-Jacobi-preconditioned GMRES(restart); lam in: guess, out: solution. Returns
        (iterations, true relative residual)."""
        _f64(K, E, lam)
        it, rr = ctypes.c_int(), ctypes.c_double()
        self._check(self._L.hdg_skeleton_solve(self._h, _ptr(K), _ptr(E), _ptr(lam), float(rtol), int(maxit),
                                               int(restart), ctypes.byref(it), ctypes.byref(rr), _stream(stream)),
                    "hdg_skeleton_solve")
        return it.value, rr.value

    # ---- saved local solutions: SURVEY.md §8(f) NEXT #2, PAPER.md:359 ------------------------------------------------
    def condense_assemble(self, A, B, C, D, r_e, r_f, K, E, factors, info, stream=None):
        """Fused condensation + skeleton assembly (single rank): S_e, g_e go straight into K, E (bitwise equal to
        condense + assemble_skeleton)."""
        _f64(A, B, C, D, r_e, r_f, K, E)
        self._check(self._L.hdg_condense_assemble(self._h, *map(_ptr, (A, B, C, D, r_e, r_f, K, E, factors, info)),
                                                  _stream(stream)), "hdg_condense_assemble")

    def skeleton_structure(self, row_ptr=None, col_idx=None, blk_off=None, stream=None):
        self._check(self._L.hdg_skeleton_structure(self._h, *map(_ptr, (row_ptr, col_idx, blk_off)), _stream(stream)),
                    "hdg_skeleton_structure")

    def condense_saved(self, A, B, C, D, r_e, r_f, S, g, factors, X, info, stream=None):
        """hdg_condense that also saves X_e = A_e^-1 [B_e | r_e] (written by the kernels that form it)."""
        _f64(A, B, C, D, r_e, r_f, S, g, X)
        self._check(self._L.hdg_condense_saved(self._h, *map(_ptr, (A, B, C, D, r_e, r_f, S, g, factors, X, info)),
                                               _stream(stream)), "hdg_condense_saved")

    def save_solutions(self, factors, B, r_e, X, stream=None):
        """X_e = A_e^-1 [B_e | r_e] (n_e x (n_f + 1) row-major per element) from the saved factors."""
        _f64(B, r_e, X)
        self._check(self._L.hdg_save_solutions(self._h, *map(_ptr, (factors, B, r_e, X)), _stream(stream)),
                    "hdg_save_solutions")

    def backsubstitute_saved(self, X, lam, u, stream=None):
        """u_e = y_e - X_e[:, :n_f] lambda_e from the saved solutions (a GEMV per element)."""
        _f64(X, lam, u)
        self._check(self._L.hdg_backsubstitute_saved(self._h, _ptr(X), _ptr(lam), _ptr(u), _stream(stream)),
                    "hdg_backsubstitute_saved")

    # ---- adjoint (transposed) path: SURVEY.md §8(f) NEXT #1, PAPER.md:414-436 ---------------------------------------
    def condense_adjoint_rhs(self, factors, B, rt_e, rt_f, gt, stream=None):
        """g~_e = r~_f - B_e^T A_e^-T r~_e (rt_f None: r~_f = 0, H~ = 0)."""
        _f64(B, rt_e, gt)
        self._check(self._L.hdg_condense_adjoint_rhs(self._h, *map(_ptr, (factors, B, rt_e, rt_f, gt)),
                                                     _stream(stream)), "hdg_condense_adjoint_rhs")

    def assemble_adjoint(self, S, gt, Kt, Et, send=None, stream=None):
        """Kt = sum_e S_e^T (= K^T), Et = sum_e g~_e (send: contributions to other ranks' rows)."""
        _f64(S, gt, Kt, Et, send)
        self._check(self._L.hdg_assemble_adjoint(self._h, *map(_ptr, (S, gt, Kt, Et, send)), _stream(stream)),
                    "hdg_assemble_adjoint")

    def backsubstitute_adjoint(self, factors, C, rt_e, lam_t, ut, stream=None):
        """u~_e = A_e^-T (r~_e - C_e^T lambda~_e)."""
        _f64(C, rt_e, lam_t, ut)
        self._check(self._L.hdg_backsubstitute_adjoint(self._h, *map(_ptr, (factors, C, rt_e, lam_t, ut)),
                                                       _stream(stream)), "hdg_backsubstitute_adjoint")

    def first_error(self, info, stream=None):
        e = ctypes.c_int64()
        c = ctypes.c_int32()
        st = self._L.hdg_first_error(self._h, _ptr(info), ctypes.byref(e), ctypes.byref(c), _stream(stream))
        if st not in (HDG_OK, HDG_ERR_SINGULAR):
            self._check(st, "hdg_first_error")
        return e.value, c.value

    def debug_set_trace(self, buf):
        """Instrumentation: record clock64 stamps of CTA 0 into the int64 CUDA tensor buf (None = off)."""
        self._check(self._L.hdg_debug_set_trace(self._h, _ptr(buf)), "hdg_debug_set_trace")

    def launch_count(self) -> int:
        return int(self._L.hdg_launch_count(self._h))


def exchange_layout(elem_face, face_elem, face_ndof, elem_ndof, rank_elem_begin, rank: int):
    """a7 exchange layout of `rank`'s slab (hdg_exchange_layout: host only, no device or context needed).
    Returns dict(send_counts, send_displs, recv_counts, recv_displs [nranks] int64, send_items, recv_items [n, 3]
    int64) — see include/hdg.h for the packing."""
    L = lib()
    ef = np.ascontiguousarray(elem_face, dtype=np.int32)
    fe = np.ascontiguousarray(face_elem, dtype=np.int32)
    fn = np.ascontiguousarray(face_ndof, dtype=np.int32)
    en = np.ascontiguousarray(elem_ndof, dtype=np.int32)
    rb = np.ascontiguousarray(rank_elem_begin, dtype=np.int64)
    nranks = len(rb) - 1
    m = _Mesh(ef.shape[0], fe.shape[0], int(rb[rank]), int(rb[rank + 1] - rb[rank]), ef.ctypes.data, fe.ctypes.data,
              fn.ctypes.data, en.ctypes.data, rb.ctypes.data)
    arrs = [np.zeros(nranks, dtype=np.int64) for _ in range(4)]
    ns, nr = ctypes.c_int64(), ctypes.c_int64()
    P = ctypes.c_void_p
    st = L.hdg_exchange_layout(ctypes.byref(m), rank, nranks, *[P(a.ctypes.data) for a in arrs], ctypes.byref(ns), None,
                               ctypes.byref(nr), None)
    if st != HDG_OK:
        raise HDGError(st, "hdg_exchange_layout")
    si = np.zeros((ns.value, 3), dtype=np.int64)
    ri = np.zeros((nr.value, 3), dtype=np.int64)
    st = L.hdg_exchange_layout(ctypes.byref(m), rank, nranks, *[P(a.ctypes.data) for a in arrs], ctypes.byref(ns),
                               P(si.ctypes.data), ctypes.byref(nr), P(ri.ctypes.data))
    if st != HDG_OK:
        raise HDGError(st, "hdg_exchange_layout")
    return dict(send_counts=arrs[0], send_displs=arrs[1], recv_counts=arrs[2], recv_displs=arrs[3], send_items=si,
                recv_items=ri)


def nnz_counts(elem_face, face_elem, face_ndof, dg_ndof):
    """hdg_nnz_counts (host only): (nonzeros of the DG system matrix, nonzeros of the HDG skeleton matrix K) for the
    mesh; dg_ndof[e] = m n(p_e) DG unknowns per element (§8(f) NEXT #4, Tables 1-4)."""
    L = lib()
    ef = np.ascontiguousarray(elem_face, dtype=np.int32)
    fe = np.ascontiguousarray(face_elem, dtype=np.int32)
    fn = np.ascontiguousarray(face_ndof, dtype=np.int32)
    dn = np.ascontiguousarray(dg_ndof, dtype=np.int32)
    m = _Mesh(ef.shape[0], fe.shape[0], 0, ef.shape[0], ef.ctypes.data, fe.ctypes.data, fn.ctypes.data,
              dn.ctypes.data, None)
    a, b = ctypes.c_int64(), ctypes.c_int64()
    st = L.hdg_nnz_counts(ctypes.byref(m), dn.ctypes.data, ctypes.byref(a), ctypes.byref(b))
    if st != HDG_OK:
        raise HDGError(st, "hdg_nnz_counts")
    return a.value, b.value


def exchange_buffers(send, recv, send_counts, send_displs, recv_counts, recv_displs, rank: int, nranks: int,
                     group=None):
    """a7 transport: point-to-point torch.distributed ops moving each peer's slice of the packed send buffer to
    it and filling recv (NCCL over NVLink for CUDA tensors; gloo for CPU tensors in the multi-process tests).
    Plumbing only — packing and the ordered accumulation are libhdg kernels."""
    import torch.distributed as dist
    ops = []
    for r in range(nranks):
        if r == rank:
            continue
        if recv_counts[r] > 0:
            ops.append(dist.P2POp(dist.irecv, recv[recv_displs[r]:recv_displs[r] + recv_counts[r]], r, group))
        if send_counts[r] > 0:
            ops.append(dist.P2POp(dist.isend, send[send_displs[r]:send_displs[r] + send_counts[r]], r, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def exchange(ctx: Context, send, recv, group=None, stream=None):
    """a7 transport for a planned context without its own communicator (counts from hdg_exchange_counts), issued
    on `stream` (torch's NCCL ops order themselves after, and the stream after, the current stream). A context
    with an NCCL communicator exchanges inside hdg_assemble_* and this is a no-op."""
    if ctx.has_comm:
        return
    import torch
    sc, sd, rc, rd = ctx.exchange_counts()
    if stream is not None and send is not None and send.is_cuda:
        with torch.cuda.stream(stream):
            exchange_buffers(send, recv, sc, sd, rc, rd, ctx.rank, ctx.nranks, group)
    else:
        exchange_buffers(send, recv, sc, sd, rc, rd, ctx.rank, ctx.nranks, group)


def nccl_context(device: int, rank: int, nranks: int, group=None) -> Context:
    """Context with its own NCCL communicator, bootstrapped over an initialised torch.distributed group: rank 0
    draws the id (hdg_get_unique_id) and broadcasts it (plumbing only)."""
    import torch.distributed as dist
    obj = [get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return Context(device, rank, nranks, nccl_id=obj[0])
