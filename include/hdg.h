/* include/hdg.h — C ABI of libhdg: element-local static condensation and its inverse on B200 (sm_100a), fp64.
 *
 * The operations are those of the paper's hybridization (§3.4):
 * the linearised HDG system Eq. 44 [[A B R],[C D S],[L M N]] [dQ dW dL] = [F G H] is split into
 * element-local equations (Eq. ls) and the trace equations (Eq. cons);
 * eliminating the element unknowns yields the hybridized system K dL = E (Eq. hybridsystem).
 * The local matrix is block-diagonal by element, so everything is element-wise.
 *
 * Notation: per element e,
 *   A_e  (n_e x n_e)  = [[A,B],[C,D]] restricted to e          (paper's local matrix)
 *   B_e  (n_e x n_f)  = [R;S] restricted to e's rows, e's trace columns
 *   C_e  (n_f x n_e)  = [L M] restricted to e's trace rows, e's columns
 *   D_e  (n_f x n_f)  = e's contribution to N
 *   r_e  (n_e), r_f (n_f) = [F;G]|_e and e's contribution to H
 *   S_e = D_e - C_e A_e^-1 B_e,  g_e = r_f - C_e A_e^-1 r_e       (e's contributions to K and E)
 *   u_e = A_e^-1 (r_e - B_e lambda_e)                            (reconstruction, Eq. ls)
 * n_e = element unknowns, n_f = sum over the element's three face slots of the face's trace size (0 for a slot
 * of -1). Trace columns/rows of an element are ordered slot 0, 1, 2, each face's dofs contiguous, in the face's
 * global dof order.
 *
 * Memory conventions:
 *   - All array arguments of the compute calls are CUDA DEVICE pointers owned by the caller, except where
 *     marked [host]. The library allocates only its own context/plan workspace (freed by hdg_ctx_destroy).
 *   - Element blocks are row-major and packed densely in local element order, without gaps: block X of local
 *     element l starts at sum_{l' < l} size_X(l') doubles (size_A = n_e^2, size_B = n_e n_f, size_C = n_f n_e,
 *     size_D = n_f^2, size_re = n_e, size_rf = n_f, size_S = n_f^2, size_g = n_f, size_u = n_e).
 *     Every base pointer must be 16-byte aligned. hdg_plan reports each array's total length.
 *   - lambda and E are indexed by trace dof: face f's dofs occupy [face_off[f], face_off[f] + face_ndof[f]),
 *     face_off = exclusive prefix sum of face_ndof over global face ids.
 *   - Every compute call is stream-ordered and asynchronous on the given stream; argument errors are detected
 *     synchronously before any launch and return HDG_ERR_ARG with nothing launched.
 *   - Threading: a context is used by one host thread at a time; one context per device.
 *   - Errors: hdg_status codes, never exceptions; hdg_last_error(ctx) holds a message for the last failure.
 *     Numerical failure is reported per element in info[] (LAPACK getrf convention), see hdg_condense.
 */
#ifndef HDG_H
#define HDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hdg_ctx_s* hdg_ctx;
typedef void* hdg_stream; /* a cudaStream_t (NULL = legacy default stream) */

typedef enum {
  HDG_OK = 0,
  HDG_ERR_ARG = 1,         /* bad argument / shape / alignment; nothing launched */
  HDG_ERR_SINGULAR = 2,    /* hdg_first_error found an element with info != 0 */
  HDG_ERR_CUDA = 3,        /* CUDA runtime error (message in hdg_last_error) */
  HDG_ERR_NOMEM = 4,       /* workspace allocation failed */
  HDG_ERR_STATE = 5,       /* call out of order (e.g. compute before hdg_plan) */
  HDG_ERR_UNSUPPORTED = 6, /* sizes outside what this build supports (n_e > 256, n_f > 96, ...) */
  HDG_ERR_NCCL = 7         /* NCCL unavailable or an NCCL call failed (message in hdg_last_error / stderr) */
} hdg_status;

/* Library version and the supported maxima. */
const char* hdg_version(void);
int hdg_max_elem_ndof(void);   /* largest n_e supported by the condensation kernels */
int hdg_max_face_ndof(void);   /* largest n_f (element trace size) supported */

const char* hdg_status_string(hdg_status s);

/* a7 bootstrap: a fresh NCCL unique id ([host] 128 bytes), generated on ONE rank (rank 0) and
 * distributed to the others by the caller (e.g. torch.distributed broadcast). NCCL is loaded at run time
 * (libnccl.so.2); HDG_ERR_NCCL if it is unavailable. */
hdg_status hdg_get_unique_id(unsigned char id[128]);

/* Context on CUDA device `device` for rank `rank` of `nranks` (element-slab partition; see hdg_mesh).
 * [host] out. The context owns the plan and all workspace.
 * nccl_id [host, 128 bytes]: NULL for a single rank, or for nranks > 1 when the caller transports the exchange
 * buffers itself (hdg_exchange_counts / hdg_skeleton_accumulate). Non-NULL: every rank passes the same id from
 * hdg_get_unique_id and the call creates the context's NCCL communicator (ncclCommInitRank: collective, blocks
 * until all nranks ranks have called it); hdg_assemble_skeleton / hdg_assemble_adjoint then perform the
 * shared-face exchange themselves, stream-ordered. Errors: HDG_ERR_ARG (bad rank/nranks), HDG_ERR_CUDA (device),
 * HDG_ERR_UNSUPPORTED (not compute capability 10.x), HDG_ERR_NCCL (communicator). */
hdg_status hdg_ctx_create(hdg_ctx* out, int device, int rank, int nranks, const unsigned char* nccl_id);
/* 1 if the context owns an NCCL communicator (created with an id), else 0. */
int hdg_ctx_has_comm(hdg_ctx ctx);
void hdg_ctx_destroy(hdg_ctx ctx);
const char* hdg_last_error(hdg_ctx ctx);

/* The mesh skeleton and degree map (§3.1): all pointers [host], global ids throughout.
 * Faces are the element edges carrying trace unknowns; a slot of -1 carries none (e.g. the paper's boundary
 * edges). This rank owns elements [elem_begin, elem_begin + n_elem). A face row of K is
 * owned by the rank of its left (lower-id) element; owned faces must form a contiguous id range. */
typedef struct {
  int64_t n_elem_global;     /* E */
  int64_t n_face;            /* F */
  int64_t elem_begin;        /* first element of this rank's slab */
  int64_t n_elem;            /* elements of this rank's slab */
  const int32_t* elem_face;  /* [E][3] face id per slot, or -1 */
  const int32_t* face_elem;  /* [F][2] (left, right), left < right; right = -1 for a one-sided face */
  const int32_t* face_ndof;  /* [F] trace dofs of the face, m (p_f + 1) */
  const int32_t* elem_ndof;  /* [E] n_e of each element */
  const int64_t* rank_elem_begin; /* [nranks + 1] slab boundaries (NULL iff nranks == 1) */
} hdg_mesh;

typedef struct {
  int64_t n_elem;                       /* local elements */
  int64_t len_A, len_B, len_C, len_D;   /* doubles of each packed input array */
  int64_t len_re, len_rf;
  int64_t len_S, len_g, len_u;          /* doubles of each packed output array */
  int64_t factor_bytes;                 /* size of the opaque factor buffer */
  int64_t owned_face_begin, n_owned_faces;   /* rows of K stored on this rank */
  int64_t nnzb;                         /* blocks in the owned rows (col_idx length) */
  int64_t nvals;                        /* doubles of K (blk_off[nnzb]) */
  int64_t owned_trace_begin, n_owned_trace;  /* E covers trace dofs [begin, begin + n) */
  int64_t n_trace;                      /* global trace dofs (length of lambda) */
  int32_t n_buckets;                    /* distinct (n_e, n_f) classes among local elements */
  int32_t max_ne, max_nf;
  int64_t send_doubles, recv_doubles;   /* exchange buffer sizes (0 when nranks == 1) */
  int64_t len_X;                        /* doubles of the saved local solutions (hdg_save_solutions) */
} hdg_plan_info;

/* a0 plan (once per mesh and degree map): validates the mesh, buckets local elements by (n_e, n_f) (the hp
 * degree classes), computes packed offsets, builds the block-CSR structure of the owned skeleton rows on the
 * device (row_ptr/col_idx/blk_off) and the exchange lists for faces shared between slabs.
 * Synchronizes `stream`. Replaces any previous plan of the context. [host] info. */
hdg_status hdg_plan(hdg_ctx ctx, const hdg_mesh* mesh, hdg_plan_info* info, hdg_stream stream);

/* a1-a5 condensation (Eq. hybridsystem): for every local element, factor A_e with partial
 * pivoting and form S_e = D_e - C_e A_e^-1 B_e, g_e = r_f - C_e A_e^-1 r_e.
 * Inputs A, B, C, D, r_e, r_f: packed as above (read only). Outputs S, g: packed. factors: opaque buffer of
 * plan.factor_bytes bytes holding the element factorizations for hdg_backsubstitute ("can be saved ... and
 * reused during the reconstruction"); its per-element records are 128-byte multiples, so a 128-byte
 * aligned buffer (any cudaMalloc / torch allocation) keeps every record on whole DRAM atoms. info: int32 [n_elem]; info[l] = 0 on success, or k+1 if
 * the k-th pivot of element l was exactly zero, in which case S_l and g_l are set to NaN. */
hdg_status hdg_condense(hdg_ctx ctx, const double* A, const double* B, const double* C, const double* D,
                        const double* r_e, const double* r_f, double* S, double* g, void* factors,
                        int32_t* info, hdg_stream stream);

/* Re-condensation with a diagonal shift (§8(f) NEXT #4): the pseudo-time relaxation adds <phi_h, dw_h / dt> to
 * the linearised system (backward Euler in an artificial time, local time step dt_K per element),
 * i.e. M_e / dt_K on the element's w unknowns. With an orthonormal (modal) basis M_e = |K| I, so the term is the
 * diagonal shift |K| / dt_K = (lambda_c + 4 lambda_v) / CFL^n on those unknowns (0 on q). This call condenses
 * A_e + diag(shift_e) exactly as hdg_condense condenses A_e — the shift is added while the kernels stage A_e (no
 * extra pass over A in HBM), so every Newton step re-condenses the changed matrix at the cost of hdg_condense.
 * shift: device, packed like r_e (n_e doubles per element, 16-byte aligned), read only. Everything else, including
 * info and the saved factors (of the shifted matrix), as hdg_condense. */
hdg_status hdg_condense_shifted(hdg_ctx ctx, const double* A, const double* B, const double* C, const double* D,
                                const double* r_e, const double* r_f, const double* shift, double* S, double* g,
                                void* factors, int32_t* info, hdg_stream stream);

/* Fused condensation and assembly (§8(f) NEXT #2): as hdg_condense followed by hdg_assemble_skeleton, but S_e and
 * g_e never reach HBM — the condensation kernels add them into K and E from their registers / shared memory
 * (fp64 atomics). Every entry of K and E has at most two contributions (the left and the right element of its
 * face), and (0 + a) + b == (0 + b) + a in IEEE arithmetic, so K and E are bitwise those of the ordered
 * left-then-right gather. K [plan.nvals], E [plan.n_owned_trace]: device outputs, zeroed by the call
 * first; factors and info as for hdg_condense (S and g are not produced: the adjoint assembly needs hdg_condense).
 * Single rank (HDG_ERR_UNSUPPORTED otherwise: shared-face rows need the exchange). The block-CSR structure of K is
 * the plan's (hdg_skeleton_structure). */
hdg_status hdg_condense_assemble(hdg_ctx ctx, const double* A, const double* B, const double* C, const double* D,
                                 const double* r_e, const double* r_f, double* K, double* E, void* factors,
                                 int32_t* info, hdg_stream stream);

/* Copy the plan's block-CSR structure of the owned rows (as hdg_assemble_skeleton does): row_ptr [n_owned_faces+1],
 * col_idx [nnzb], blk_off [nnzb+1] (device; any may be NULL). Stream-ordered. */
hdg_status hdg_skeleton_structure(hdg_ctx ctx, int32_t* row_ptr, int32_t* col_idx, int64_t* blk_off,
                                  hdg_stream stream);

/* a6 (+a7 pack) assembly of the owned skeleton rows: K[f, f'] = sum over local elements e adjacent to both of
 * S_e[slot(f), slot(f')], E[f] = sum of g_e[slot(f)], contributions taken left (lower element id) then right
 * (SURVEY.md S10). Block-CSR over owned rows: row_ptr [n_owned_faces + 1] int32 (block
 * counts, 0-based), col_idx [nnzb] int32 global face ids ascending (diagonal included), blk_off [nnzb + 1]
 * int64 offsets of each row-major n_fp(row) x n_fp(col) block in K (doubles), K [nvals], E [n_owned_trace].
 * row_ptr/col_idx/blk_off may be NULL (structure not copied out; it is fixed by the plan).
 * a7, nranks > 1: the right (non-owner) element's contributions to a shared face row travel to
 * the row's owner and are added AFTER the owner's own, so K and E are bitwise those of one rank (P12).
 *   - context with an NCCL communicator: this call packs them into library-owned buffers, exchanges them with
 *     one grouped ncclSend/ncclRecv on `stream` and accumulates them, all stream-ordered (no host sync); `send`
 *     is ignored (may be NULL).
 *   - context without one: send (device, plan.send_doubles) receives this rank's contributions to face rows
 *     owned by other ranks; the caller exchanges it with hdg_exchange_counts' layout (on the same stream order)
 *     and finishes with hdg_skeleton_accumulate. */
hdg_status hdg_assemble_skeleton(hdg_ctx ctx, const double* S, const double* g, int32_t* row_ptr,
                                 int32_t* col_idx, int64_t* blk_off, double* K, double* E, double* send,
                                 hdg_stream stream);

/* a7 exchange layout: per peer rank, doubles sent/received and their offsets in send/recv [host, nranks]. */
hdg_status hdg_exchange_counts(hdg_ctx ctx, int64_t* send_counts, int64_t* send_displs, int64_t* recv_counts,
                               int64_t* recv_displs);

/* a7 exchange layout, host only (no device, no context: usable for planning and by CPU tests of the multi-rank
 * path). All pointers [host]. mesh: as for hdg_plan, rank_elem_begin required. Per peer rank (arrays of nranks):
 * doubles sent/received and their offsets in the packed buffers (same values hdg_exchange_counts reports after
 * hdg_plan). Items, [n][3] int64 each, NULL to query the counts only:
 *   send_items: (global face f, LOCAL element l, offset o): send[o .. o + n_fp) = g_l[slot f], then the
 *               n_fp x n_f(l) strip S_l[slot f rows, all columns] row-major — face f's row is owned by the rank
 *               of its left element, which is remote;
 *   recv_items: (owned face f, GLOBAL remote element e, offset o), same packing, added after the owner's own
 *               contribution by hdg_skeleton_accumulate (left, then right).
 * Items are grouped by peer rank, then face id. Returns HDG_ERR_ARG on inconsistent arguments. */
hdg_status hdg_exchange_layout(const hdg_mesh* mesh, int rank, int nranks, int64_t* send_counts, int64_t* send_displs,
                               int64_t* recv_counts, int64_t* recv_displs, int64_t* n_send_items, int64_t* send_items,
                               int64_t* n_recv_items, int64_t* recv_items);

/* a7 finish: add the contributions received from other ranks (recv, device, plan.recv_doubles) into the owned
 * rows, after this rank's own (left) contributions: the result is bitwise identical to one rank. */
hdg_status hdg_skeleton_accumulate(hdg_ctx ctx, const double* recv, double* K, double* E, hdg_stream stream);

/* a8 back-substitution (Eq. ls): u_e = A_e^-1 (r_e - B_e lambda_e) for every local
 * element, with lambda_e gathered from the global trace vector lambda [n_trace] (device) in slot order.
 * factors: from hdg_condense on the same plan. B, r_e: the packed inputs of hdg_condense. u: packed output. */
hdg_status hdg_backsubstitute(hdg_ctx ctx, const void* factors, const double* B, const double* r_e,
                              const double* lambda, double* u, hdg_stream stream);

/* ---- saved local solutions: SURVEY.md §8(f) NEXT #2 ----------------------------------------------------------
 * "the solutions to Eq. (ls) can be saved after the assembly of the hybridized system and reused during the
 * reconstruction". X_e = A_e^-1 [B_e | r_e]: n_e x (n_f + 1) row-major per element, packed densely
 * in local element order (plan.len_X doubles in total); its last column is y_e = A_e^-1 r_e. */

/* X_e = A_e^-1 [B_e | r_e] for every local element from the saved factors (P A_e = L U: permute, forward, backward
 * solves of the n_f + 1 right-hand sides on the FP64 tensor cores). factors, B, r_e: as for hdg_backsubstitute.
 * X: device output (plan.len_X doubles, 16-byte aligned). */
hdg_status hdg_save_solutions(hdg_ctx ctx, const void* factors, const double* B, const double* r_e, double* X,
                              hdg_stream stream);

/* hdg_condense that also saves the local solutions X (as hdg_save_solutions would): the condensation kernels that
 * form X = A_e^-1 [B_e | r_e] on the way to S_e (the warp-per-element kernel, n_e <= 32, and the panel kernel)
 * write it from shared memory; for the buckets whose kernels never form it (the sweep kernels eliminate the C rows
 * alongside A instead) the save pass runs on the fresh factors. Arguments as hdg_condense plus X (device,
 * plan.len_X doubles). */
hdg_status hdg_condense_saved(hdg_ctx ctx, const double* A, const double* B, const double* C, const double* D,
                              const double* r_e, const double* r_f, double* S, double* g, void* factors, double* X,
                              int32_t* info, hdg_stream stream);

/* Reconstruction from the saved solutions: u_e = y_e - X_e[:, 0:n_f] lambda_e (= A_e^-1 (r_e - B_e lambda_e)),
 * a GEMV per element reading n_e (n_f + 1) doubles instead of the factors, B_e and r_e. lambda as for
 * hdg_backsubstitute; u packed like hdg_backsubstitute's. */
hdg_status hdg_backsubstitute_saved(hdg_ctx ctx, const double* X, const double* lambda, double* u, hdg_stream stream);

/* ---- the skeleton solve: SURVEY.md §8(f) NEXT #3 ---------------------------------------------------------------
 * "First, the hybridized system is assembled and then being solved for dLambda"; the paper uses an
 * ILU(n)-preconditioned GMRES from PETSc. Here: restarted GMRES(restart), right-preconditioned
 * with block Jacobi (the inverses of K's diagonal face blocks), all vector work in libhdg's kernels, deterministic
 * reductions. Single rank (nranks == 1; HDG_ERR_UNSUPPORTED otherwise) and face trace sizes <= 24. */

/* y = K x over the owned rows: x device [n_trace] (global trace numbering), y device [n_owned_trace]; K as filled by
 * hdg_assemble_skeleton on this plan. Stream-ordered. */
hdg_status hdg_skeleton_spmv(hdg_ctx ctx, const double* K, const double* x, double* y, hdg_stream stream);

/* Solve K lambda = E: lambda device [n_trace], in: initial guess, out: the solution. Stops when the relative
 * residual ||E - K lambda|| / ||E|| <= rtol (Arnoldi estimate; the true residual of the returned lambda is written
 * to relres [host]) or after maxit iterations (iters [host]). Synchronizes the stream (the Hessenberg system lives on
 * the host); the workspace ((restart + 1) n_trace doubles + the block inverses) is kept in the plan. */
hdg_status hdg_skeleton_solve(hdg_ctx ctx, const double* K, const double* E, double* lambda, double rtol, int maxit,
                              int restart, int* iters, double* relres, hdg_stream stream);

/* ---- adjoint (transposed) use of the same factors: SURVEY.md §8(f) NEXT #1, PAPER.md:414-436 ----------------
 * The adjoint local matrix is the transpose of the primal one and the hybridized adjoint matrix
 * is K^T, so the adjoint reuses the plan and the factors of hdg_condense (same element degrees). */

/* Adjoint right-hand side, element part of E~ = -[R^T S^T][[A B][C D]]^-T [F~; G~]:
 * g~_e = r~_f - B_e^T A_e^-T r~_e for every local element. factors, B: as for hdg_backsubstitute. rt_e: packed
 * like r_e; rt_f: packed like r_f, or NULL for r~_f = 0 (H~ = 0). gt: packed like g (output).
 * All device pointers, 16-byte aligned. */
hdg_status hdg_condense_adjoint_rhs(hdg_ctx ctx, const void* factors, const double* B, const double* rt_e,
                                    const double* rt_f, double* gt, hdg_stream stream);

/* Adjoint skeleton assembly: Kt = sum_e S_e^T (= K^T block by block) into the plan's block-CSR
 * structure (same row_ptr / col_idx / blk_off as hdg_assemble_skeleton), Et = sum_e g~_e, left then right.
 * S from hdg_condense, gt from hdg_condense_adjoint_rhs. With nranks > 1 the exchange is as for
 * hdg_assemble_skeleton: inside the call when the context has an NCCL communicator; otherwise send
 * (plan.send_doubles, device) receives this rank's contributions to rows owned by others (strips of S_e^T, same
 * layout) and, after the caller's transport, hdg_skeleton_accumulate(recv, Kt, Et) finishes the owned rows
 * (bitwise as one rank). */
hdg_status hdg_assemble_adjoint(hdg_ctx ctx, const double* S, const double* gt, double* Kt, double* Et,
                                double* send, hdg_stream stream);

/* Adjoint reconstruction: u~_e = A_e^-T (r~_e - C_e^T lambda~_e), lambda~_e gathered from the
 * adjoint trace vector lambda_t [n_trace] in slot order. C: the packed input of hdg_condense. ut: packed like u. */
hdg_status hdg_backsubstitute_adjoint(hdg_ctx ctx, const void* factors, const double* C, const double* rt_e,
                                      const double* lambda_t, double* ut, hdg_stream stream);

/* DG-vs-HDG global-matrix size (§8(f) NEXT #4; "blocks ... O(m^2 p^2(d-1)) entries" vs DG's
 * "O(m^2 p^2d)"; the nonzero ratios of Tables 1-4). Host only (no device or context). mesh: as for hdg_plan
 * (all pointers [host]; elem_begin / n_elem / elem_ndof / rank_elem_begin unused). dg_ndof [host, E]: the DG
 * unknowns of each element, m n(p_K) with n(p) = (p+1)(p+2)/2 and m the number of equations (4 for 2D Euler /
 * Navier-Stokes: the DG scheme has no gradient unknowns). Outputs [host]:
 *   nnz_dg  = sum_K dg_ndof_K^2 + sum over faces with two elements of 2 dg_ndof_L dg_ndof_R;
 *   nnz_hdg = sum over face rows f of sum over the faces f' of f's elements of face_ndof_f face_ndof_f'
 *             (= plan.nvals of a single-rank plan: the block-CSR skeleton matrix K).
 * Returns HDG_ERR_ARG on inconsistent arguments. */
hdg_status hdg_nnz_counts(const hdg_mesh* mesh, const int32_t* dg_ndof, int64_t* nnz_dg, int64_t* nnz_hdg);

/* Lowest local element with info != 0 (synchronizes stream). Returns HDG_OK with *elem = -1 if none, or
 * HDG_ERR_SINGULAR with the element (local index) and its info code ("singular local block -> diagnostic
 * naming the element"). */
hdg_status hdg_first_error(hdg_ctx ctx, const int32_t* info, int64_t* elem, int32_t* code, hdg_stream stream);

/* Kernel launches issued by the last hdg_condense / hdg_assemble_skeleton(+accumulate) / hdg_backsubstitute
 * calls of this context (instrumentation for the benchmark's launch count). */
int64_t hdg_launch_count(hdg_ctx ctx);

/* Instrumentation (profiling builds/tools only): when non-NULL, hdg_condense records clock64() stamps of CTA 0
 * into the device buffer trace (>= 4 x 256 int64), see tools/trace_condense.py. NULL (default) = off. */
hdg_status hdg_debug_set_trace(hdg_ctx ctx, long long* trace);

#ifdef __cplusplus
}
#endif
#endif /* HDG_H */
