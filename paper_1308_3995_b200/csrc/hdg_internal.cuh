// hdg_internal.cuh — shared definitions of libhdg's kernels and host runtime (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/hdg.h"

namespace hdg {

constexpr int kNB = 16;          // panel width of the blocked elimination (multiple of 4 = DMMA k)
constexpr int kSweepNB = 16;     // panel width of the sweep condensation kernel (8 measured slower: 54 vs 46 ms on C4)
constexpr int kMaxNe = 256;      // largest n_e handled by the condensation / back-substitution kernels
constexpr int kMaxNf = 96;       // largest element trace size n_f
constexpr int kMaxCT = (kMaxNf + 1 + 7) / 8;   // column tiles of [S | g] in phase B

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }

// HDG_MAX_GRID (tests/tools only): caps the persistent grids of the condensation kernels, so a small mesh runs
// several elements per CTA (the pipelined paths) — e.g. under compute-sanitizer. Unset: no cap.
int64_t grid_cap(int64_t grid);

// Geometry of the per-element working matrix T = [A | 0 | B | r_e | 0] (rows padded with zeros to R8, a
// multiple of 16). Columns: A at [0, ne), B at CB = round_up(ne, 16), r_e at CB+nf, zero padding up to C8;
// row stride ldT = 4 mod 16 doubles so that DMMA A-, B- and C-fragment accesses are bank-conflict free.
struct Geo {
  int ne, nf, R8, CB, NC, C8, ldT;
  __host__ __device__ Geo(int ne_, int nf_) : ne(ne_), nf(nf_) {
    R8 = round_up(ne, 16);
    CB = R8;
    NC = CB + nf + 1;
    C8 = round_up(NC, 8);
    ldT = round_up(C8 - 4, 16) + 4;
  }
  __host__ __device__ int64_t t_doubles() const { return (int64_t)R8 * ldT; }
  // shared memory of the condensation kernel: [T (if in smem)] [U11^-1 per panel] [L11^-1] [48 doubles broadcast buffer] [2 mbarriers] [piv] [flag, spec]
  __host__ __device__ int64_t smem_bytes(bool t_in_smem) const {
    const int npan = (ne + kNB - 1) / kNB;
    return 8 * ((t_in_smem ? t_doubles() : 0) + (int64_t)(npan + 1) * kNB * 20 + 48 + 2) + 4 * (int64_t)R8 + 16;
  }
};

// Smallest row stride >= cols (doubles) that is 4 or 12 mod 16: every DMMA A/B-fragment load (8-byte, lanes
// (gid, tig) -> row gid / k tig) of a 16-lane phase then hits 32 distinct banks.
__host__ __device__ constexpr int pad_ld(int cols) {
  return (cols % 16 <= 4) ? cols - cols % 16 + 4 : (cols % 16 <= 12 ? cols - cols % 16 + 12 : cols - cols % 16 + 20);
}

// Geometry of the sweep condensation kernel (condense_sweep.cu): T = [A | 0 | B | r_e | 0] with RA = round8(n_e)
// rows (zero padding rows), B at column CB = round8(n_e), NCAB = CB + round8(n_f + 1) columns used; the C_e rows
// in a second region Cr of NF8 = round8(n_f) rows x CB columns. [S | g] is CTs = round8(n_f + 1) / 8 column tiles.
struct SweepGeo {
  int ne, nf, RA, CB, NCAB, ldT, NF8, ldC, CTs, npan, ntiles;
  __host__ __device__ SweepGeo(int ne_, int nf_) : ne(ne_), nf(nf_) {
    RA = round_up(ne, 8);
    CB = RA;
    NCAB = CB + round_up(nf + 1, 8);
    ldT = pad_ld(NCAB);
    NF8 = round_up(nf, 8);
    ldC = pad_ld(CB);
    CTs = round_up(nf + 1, 8) / 8;
    npan = (ne + kSweepNB - 1) / kSweepNB;
    ntiles = (NF8 / 8) * CTs;
  }
  // [T][Cr][L11^-1 x2][U11^-1 x2][2 broadcast slots of 40] doubles, 4 mbarriers, piv[RA], fail flag (+pad)
  __host__ __device__ int64_t smem_bytes() const {
    return 8 * ((int64_t)RA * ldT + (int64_t)NF8 * ldC + 4 * kNB * 20 + 80) + 8 * 4 + 4 * (int64_t)RA + 16;
  }
};

// Opaque per-element factor record: [LU of P A_e, row-major, ne*ne doubles][perm: ne int32][pad to 128 B];
// perm[i] = the row of A_e that is row i of P A_e. Records start on 128-byte boundaries (of a 128-byte aligned
// buffer): with 16-byte padding every other C4 record (115,680 B) started 32 B into a 64-byte DRAM atom, so the
// solves' 128-byte row segments touched three atoms instead of two (ncu: the adjoint kernels read 1.25x their
// algorithmic bytes)
__host__ __device__ inline int64_t factor_bytes(int ne) { return ((int64_t)ne * ne * 8 + (int64_t)ne * 4 + 127) / 128 * 128; }

struct CondenseArgs {
  const double *A, *B, *C, *D, *re, *rf;
  const double* shift;    // NULL, or per-element diagonal shift packed like r_e: A_e + diag(shift_e) is condensed
  double *S, *g;
  unsigned char* factors;
  int32_t* info;
  const int32_t* elems;   // local element ids of this bucket
  const int64_t *offA, *offB, *offC, *offD, *offRe, *offRf, *offS, *offG, *offF;
  int ne, nf;
  int64_t count;
  double* scratch;        // global workspace for T when it does not fit in shared memory
  long long* trace;       // instrumentation: clock64 stamps of CTA 0 (NULL = off)
  int debug;              // profiling experiments only (HDG_DEBUG_MODE): 1 = workers skip their MMA work, 2 = skip the [S|g] MMAs,
                          // 8 = sweep [S|g] tiles round-robin instead of the row map (A/B); bits 8-13 = the helper warp's
                          // share of the trailing blocks in 64ths (0 = kHelperShare, 1 = the interleaved deal);
                          // bit 26 = the next element's last rows / C rows issued after barrier E, bit 27 = its accumulators
                          // loaded at its start (the round-2 forms, A/B); panel kernel: 32 = factor rows by a warp copy
                          // loop instead of TMA bulk stores, 64 = two [S|g] items per warp pass, 128 = with shared B fragments
  // fused condense -> assemble (hdg_condense_assemble, §8(f) NEXT #2): when Kf != NULL, S_e and g_e go straight
  // into K and E by fp64 atomics instead of being stored — every K / E entry has at most two contributions (left
  // and right element of a face) and (0 + a) + b = (0 + b) + a in IEEE arithmetic, so the result is bitwise the
  // ordered gather's (left then right, R9)
  double* Kf;
  double* Ef;
  const int64_t* eblk;    // [n][9] K offset of block (slot a, slot b) of local element l (-1: row not owned)
  const int64_t* eE;      // [n][3] E offset of slot a's first dof (-1: not owned)
  const int32_t* eslot;   // [n][4] slot start rows in S_e: 0, n0, n0 + n1, n_f
  double* Xout;           // NULL, or the saved local solutions X_e = A_e^-1 [B_e | r_e] (n_e x (n_f+1), at offX)
  const int64_t* offX;
  int32_t* redo;          // row-tile kernel: elements whose GEPP speculation failed (redone on the exact path)
  int32_t* redo_count;
  int32_t* mark;          // [n] per-element failed-speculation marks (zero between calls)
};

// S_e / g_e output of a condensation kernel for one element: stored at S, g, or (fused mode, Kf != NULL) scattered
// into K / E through the element's block-offset table
struct SgDst {
  double* S;             // S_e (NULL in the fused mode)
  double* g;
  double* Kf;
  double* Ef;
  const int64_t* eblk;   // [9] this element's block offsets in K (-1: row not owned)
  const int64_t* eE;     // [3]
  const int32_t* so;     // [4] slot start rows
};
__device__ __forceinline__ SgDst sg_dst(const CondenseArgs& a, int64_t l) {
  SgDst d;
  d.Kf = a.Kf;
  d.Ef = a.Ef;
  if (a.Kf) {
    d.S = nullptr;
    d.g = nullptr;
    d.eblk = a.eblk + 9 * l;
    d.eE = a.eE + 3 * l;
    d.so = a.eslot + 4 * l;
  } else {
    d.S = a.S + a.offS[l];
    d.g = a.g + a.offG[l];
    d.eblk = nullptr;
    d.eE = nullptr;
    d.so = nullptr;
  }
  return d;
}
__device__ __forceinline__ int fused_slot(const int32_t* so, int r) { return r >= so[1] ? (r >= so[2] ? 2 : 1) : 0; }
// S_e[row][c .. c+1] (c even: both in one face slot, face trace sizes are even)
__device__ __forceinline__ void out_S2(const SgDst& d, int nf, int row, int c, double v0, double v1) {
  if (!d.Kf) {
    *reinterpret_cast<double2*>(d.S + (int64_t)row * nf + c) = make_double2(v0, v1);
    return;
  }
  const int sa = fused_slot(d.so, row), sb = fused_slot(d.so, c);
  const int64_t base = d.eblk[3 * sa + sb];
  if (base < 0) return;
  double* q = d.Kf + base + (int64_t)(row - d.so[sa]) * (d.so[sb + 1] - d.so[sb]) + (c - d.so[sb]);
  atomicAdd(q, v0);
  atomicAdd(q + 1, v1);
}
__device__ __forceinline__ void out_S1(const SgDst& d, int nf, int row, int c, double v) {
  if (!d.Kf) {
    d.S[(int64_t)row * nf + c] = v;
    return;
  }
  const int sa = fused_slot(d.so, row), sb = fused_slot(d.so, c);
  const int64_t base = d.eblk[3 * sa + sb];
  if (base >= 0) atomicAdd(d.Kf + base + (int64_t)(row - d.so[sa]) * (d.so[sb + 1] - d.so[sb]) + (c - d.so[sb]), v);
}
__device__ __forceinline__ void out_g(const SgDst& d, int row, double v) {
  if (!d.Kf) {
    d.g[row] = v;
    return;
  }
  const int sa = fused_slot(d.so, row);
  const int64_t base = d.eE[sa];
  if (base >= 0) atomicAdd(d.Ef + base + (row - d.so[sa]), v);
}

struct BacksubArgs {
  const unsigned char* factors;
  const double *B, *re, *lambda;
  double* u;
  const int32_t* elems;
  const int64_t *offB, *offRe, *offU, *offF;
  const int32_t* elem_face;   // global [E][3]
  const int32_t* face_ndof;   // global [F]
  const int64_t* face_off;    // global [F+1]
  int64_t elem_begin;
  int ne, nf;
  int64_t count;
};

// saved local solutions (§8(f) NEXT #2): X_e = A_e^-1 [B_e | r_e], n_e x (n_f + 1) row-major
struct SolutionsArgs {
  const unsigned char* factors;
  const double *B, *re, *lambda;
  double* X;          // hdg_save_solutions: output; hdg_backsubstitute_saved: input
  const double* Xin;
  double* u;
  const int32_t* elems;
  const int64_t *offB, *offRe, *offF, *offX, *offU;
  const int32_t* elem_face;
  const int32_t* face_ndof;
  const int64_t* face_off;
  int64_t elem_begin;
  int ne, nf;
  int64_t count;
};

struct AdjointArgs {
  const unsigned char* factors;
  const double *re, *rf, *M, *lambda;   // M = B_e (adjoint rhs) or C_e (adjoint reconstruction)
  double* out;                          // g~ or u~
  const int32_t* elems;
  const int64_t *offF, *offRe, *offRf, *offM, *offOut;
  const int32_t* elem_face;
  const int32_t* face_ndof;
  const int64_t* face_off;
  int64_t elem_begin;
  int ne, nf;
  int64_t count;
};

struct Bucket {
  int ne, nf;
  int64_t count;
  int32_t* d_elems;   // device list of local element ids
  bool t_in_smem;     // panel kernel: working matrix in shared memory (else global scratch)
  bool sweep;         // condensed by the sweep kernel (condense_sweep.cu)
  bool warp;          // condensed by the warp-per-element kernel (condense_warp.cu)
  bool sweep_gt;      // condensed by the sweep kernel with its working matrix in global scratch
  bool rows;          // condensed by the row-tile kernel (condense_rows.cu)
};

// Skeleton assembly data (owned rows).
struct Skeleton {
  int64_t f0 = 0, f1 = 0;          // owned face range
  int64_t nnzb = 0, nvals = 0;
  int64_t tr0 = 0, ntr = 0;         // owned trace dof range
  int32_t* d_row_ptr = nullptr;     // [nrows+1]
  int32_t* d_col_idx = nullptr;     // [nnzb]
  int64_t* d_blk_off = nullptr;     // [nnzb+1]
  int32_t* d_blk_row = nullptr;     // [nnzb] face id of the block's row
  // exchange (nranks > 1)
  std::vector<int64_t> send_counts, send_displs, recv_counts, recv_displs;
  int64_t send_doubles = 0, recv_doubles = 0;
  int64_t n_send_items = 0, n_recv_items = 0;
  int64_t* d_send_items = nullptr;  // [n][3]: face, local element, offset (doubles) in send buffer
  int64_t* d_recv_items = nullptr;  // [n][3]: face, global element, offset in recv buffer
};

// skeleton solve workspace (skeleton_solve.cu): Krylov basis, block-Jacobi inverses, reduction partials
constexpr int kMaxFaceSolve = 24;   // largest face trace size of the skeleton solve (C5: 4 (5 + 1))
struct SolverWork {
  int64_t n = -1;
  int m = 0;
  double *V = nullptr, *w = nullptr, *z = nullptr, *partial = nullptr, *h = nullptr, *Dinv = nullptr;
  int64_t* dinv_off = nullptr;
  // distributed solve (nranks > 1): the full-length work vector (owned dofs + halo), and the halo exchange lists
  // (trace-dof indices to send / receive per peer, grouped by peer, faces ascending)
  double* xfull = nullptr;
  double *hsend = nullptr, *hrecv = nullptr;
  int64_t *d_hsend_idx = nullptr, *d_hrecv_idx = nullptr;
  int64_t n_hsend = 0, n_hrecv = 0;
  std::vector<int64_t> hs_cnt, hs_dsp, hr_cnt, hr_dsp;
  bool halo_built = false;
};

struct Plan {
  bool valid = false;
  int64_t E = 0, F = 0, eb = 0, n = 0;
  int32_t *d_elem_face = nullptr, *d_face_elem = nullptr, *d_face_ndof = nullptr;
  int64_t* d_face_off = nullptr;
  int32_t *d_ne = nullptr, *d_nf = nullptr;   // local elements
  int64_t* d_off[11] = {};                     // A B C D re rf S g u F(bytes) X: [n+1] each
  std::vector<int64_t> len;                    // totals of the above
  std::vector<Bucket> buckets;
  Skeleton sk;
  double* d_scratch = nullptr;
  int64_t scratch_doubles = 0;
  SolverWork sw;
  int max_face_ndof = 0;
  // distributed skeleton solve (nranks > 1): trace-dof ranges owned by every rank, and the halo lists of this rank
  // (trace-dof indices sent to / received from each peer, grouped by peer)
  std::vector<int64_t> rank_tr0, rank_ntr;
  std::vector<int64_t> halo_send_idx, halo_recv_idx, halo_scnt, halo_sdsp, halo_rcnt, halo_rdsp;
  int64_t* d_eblk = nullptr;   // fused condense -> assemble tables (built on first use)
  int64_t* d_eE = nullptr;
  int32_t* d_eslot = nullptr;
  int32_t* d_redo = nullptr;       // [n] + count: the row-tile kernel's redo list, and its per-element marks
  int32_t* d_redo_count = nullptr;
  int32_t* d_mark = nullptr;
  double* d_send = nullptr;   // exchange buffers owned by the plan when the context has an NCCL communicator
  double* d_recv = nullptr;
  int max_ne = 0, max_nf = 0;
  int64_t n_trace = 0;
};

enum { OFF_A = 0, OFF_B, OFF_C, OFF_D, OFF_RE, OFF_RF, OFF_S, OFF_G, OFF_U, OFF_F, OFF_X, N_OFF };

}  // namespace hdg

struct hdg_ctx_s {
  int device = 0, rank = 0, nranks = 1;
  int sms = 148;
  size_t smem_optin = 0;
  std::string last_error;
  hdg::Plan plan;
  int64_t launches = 0;
  long long* trace = nullptr;
  void* nccl_comm = nullptr;   // ncclComm_t (nranks > 1 with an NCCL id): a7 runs inside hdg_assemble_*
};

// kernel launchers (defined in the .cu files); return cudaError_t of the launch
namespace hdg {
cudaError_t launch_condense(const CondenseArgs& a, bool t_in_smem, int sms, cudaStream_t s, int64_t* launches);
bool sweep_supported(int ne, int nf, size_t smem_optin);
bool warp_supported(int ne, int nf);
bool sweep_gt_supported(int ne, int nf);
cudaError_t launch_condense_sweep_gt(const CondenseArgs& a, int sms, cudaStream_t s, int64_t* launches);
cudaError_t launch_condense_warp(const CondenseArgs& a, int sms, cudaStream_t s, int64_t* launches);
cudaError_t launch_condense_sweep(const CondenseArgs& a, int sms, size_t smem_optin, cudaStream_t s, int64_t* launches);
bool rows_supported(int ne, int nf, size_t smem_optin);
cudaError_t launch_condense_rows(const CondenseArgs& a, int sms, size_t smem_optin, cudaStream_t s, int64_t* launches);
// exact path (unblocked GEPP with the warp pivot search) for the listed elements (count on the device)
cudaError_t launch_exact_list(const CondenseArgs& a, const int32_t* list, const int32_t* count, int grid, cudaStream_t s);
cudaError_t launch_backsub(const BacksubArgs& a, int sms, cudaStream_t s, int64_t* launches);
cudaError_t launch_adjoint(const AdjointArgs& a, int mode, int sms, cudaStream_t s, int64_t* launches);
cudaError_t launch_save_solutions(const SolutionsArgs& a, int sms, cudaStream_t s, int64_t* launches);
cudaError_t skeleton_gmres(const Plan& p, SolverWork& sw, const double* K, const double* E, double* x, double rtol,
                           int maxit, int m, cudaStream_t s, int* iters, double* relres, int64_t* launches,
                           void* comm = nullptr, int rank = 0, int nranks = 1, std::string* comm_err = nullptr);
cudaError_t skeleton_spmv(const Plan& p, const double* K, const double* x, double* y, cudaStream_t s,
                          int64_t* launches);
cudaError_t launch_backsub_saved(const SolutionsArgs& a, int sms, cudaStream_t s, int64_t* launches);
cudaError_t skeleton_symbolic(Plan& p, cudaStream_t s);
cudaError_t launch_assemble(const Plan& p, const double* S, const double* g, double* K, double* E, double* send,
                            cudaStream_t s, int64_t* launches, bool transposed = false);
cudaError_t launch_accumulate(const Plan& p, const double* recv, double* K, double* E, cudaStream_t s,
                              int64_t* launches);
cudaError_t launch_first_error(const int32_t* info, int64_t n, int64_t* d_out, cudaStream_t s);
// comm.cu (NCCL resolved at run time)
bool nccl_available(std::string* err);
bool nccl_unique_id(unsigned char* out, std::string* err);
bool nccl_comm_init(void** comm, int nranks, int rank, const unsigned char* id, std::string* err);
void nccl_comm_destroy(void* comm);
bool nccl_exchange(void* comm, const Plan& p, int rank, int nranks, const double* send, double* recv, cudaStream_t s,
                   std::string* err);
bool nccl_allreduce_sum(void* comm, double* buf, size_t n, cudaStream_t s, std::string* err);
bool nccl_allgatherv_inplace(void* comm, int nranks, const std::vector<int64_t>& off, const std::vector<int64_t>& cnt,
                             double* buf, cudaStream_t s, std::string* err);
bool nccl_p2p(void* comm, int rank, int nranks, const std::vector<int64_t>& scnt, const std::vector<int64_t>& sdsp,
              const double* sbuf, const std::vector<int64_t>& rcnt, const std::vector<int64_t>& rdsp, double* rbuf,
              cudaStream_t s, std::string* err);
}  // namespace hdg
