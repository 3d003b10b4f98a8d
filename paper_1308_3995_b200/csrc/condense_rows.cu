// condense_rows.cu — rows a1-a5 of the hot path: the row-tile condensation kernel, for every
// (n_e, n_f) class whose element fits (C3, C4 and C5's n_e = 36/72/120 buckets).
//
// For each element e (Eq. hybridsystem; "condense"):
//     S_e = D_e - C_e A_e^-1 B_e,   g_e = r_f - C_e A_e^-1 r_e,
// with A_e factored by Gaussian elimination with partial pivoting (speculative, R16) and
// the factorization kept for the reconstruction.
//
// Formulation: the eliminated augmented matrix M = [[A_e, B_e | r_e], [C_e, D_e | r_f]] (n_e + n_f rows) is
// processed by ROW TILES of 8 rows (one DMMA m8n8k4 row block), up-looking (row-by-row Doolittle):
//   A row tile i (rows 8i..8i+7 of [A | B r]): for k < i, L_ik = M_ik U_kk^-1 (the GEPP multipliers, checked
//       |l| <= 1), M_i,>k -= L_ik U_k,>k; then the 8x8 diagonal block is factored (L_ii U_ii, with both
//       inverses) and U_i,>i = L_ii^-1 M_i,>i is published — the U rows include the W = L^-1 P [B r] columns.
//   C row tile c (rows of [C | D r_f]): the same k loop over all A row tiles (Y_ck = M_ck U_kk^-1 are the rows of
//       C U^-1) — what is left in its [D | r_f] columns is [S_e | g_e] = [D | r_f] - Y W. No backward
//       substitution, no separate Schur GEMM: the Schur complement is the last C row tile state.
// Each row tile is ONE warp task with the tile's 8 rows (all columns) in registers (the DMMA accumulator layout);
// only the published U rows (upper triangle of A and the W columns, 8x8 tiles stored in the DMMA B-fragment
// order) live in shared memory. Tasks are claimed in increasing order (element-major) by the CTA's warps; a task
// waits only for U tiles of lower row tiles of its element (per-row progress counters, published tile by tile
// so the chain of diagonal blocks proceeds as a wavefront) and, before it writes its element's U-store slot, for
// the element that used that slot before to be complete. The lowest unfinished task never waits: no deadlock.
// Two or more elements are in flight per SM (the U-store slots overlap where the shared memory is short: C4), so
// one element's chain of diagonal factorizations overlaps another element's bulk tensor-core work.
// Pivoting: a task that sees a multiplier |l| > 1 (GEPP would interchange rows) or a bad pivot marks its element;
// the element's last task appends it to a redo list, and the exact path (unblocked GEPP with the warp-level pivot
// search, condense_sweep.cu) redoes those elements in a second launch. When no mark is set, GEPP's pivot sequence
// is the identity and this IS GEPP.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "dev_common.cuh"
#include "hdg_internal.cuh"

namespace hdg {
namespace {

constexpr int kLdL = 12;       // row stride of the per-warp L_ii^-1 (A-fragment loads bank-conflict free)
constexpr int kWScr = 264;     // doubles of per-warp scratch: LU stage 64 + pivot reciprocals 8, L^-1 8 x 12, nxt 8 x 12
constexpr int kCtrlInts = 160; // next task, fin[4], prog[4][32] (+ pad)
constexpr int kGrp = 4;        // U tiles per TRSM group / publication (the first group: 2)

struct RowGeo {
  int ne, nf, RA, TA, NCT, TC, NT;
  int64_t tiles;   // U-store tiles (64 doubles) per element
  __host__ __device__ RowGeo(int ne_, int nf_) : ne(ne_), nf(nf_) {
    RA = round_up(ne, 8);
    TA = RA / 8;
    NCT = TA + round_up(nf + 1, 8) / 8;
    TC = round_up(nf, 8) / 8;
    NT = TA + TC;
    tiles = (int64_t)TA * NCT - (int64_t)TA * (TA - 1) / 2;
  }
  // offset (doubles) of U row tile k in an element's U store: [U_kk^-1 | U_k,k+1 | ... | U_k,NCT-1]
  __host__ __device__ int row_off(int k) const { return 64 * (k * NCT - k * (k - 1) / 2); }
};

struct RowCfg {
  int D;       // disjoint slots: C rows delayed by D = NS - 1 elements
  int NS;      // U-store slots (elements in flight)
  int P;       // pool doubles
  int ovl;     // overlap mode (NS == 2): row tiles >= ovl of slot s overlap the other slot's region
  int overlap;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;\n" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}
// warp-uniform wait until *p >= v: one acquire load inline; the polling loop (hardware sleep between polls, the
// waiting warp takes no issue slots) out of line, so the many wait sites of the unrolled loops stay small
// (__any_sync: the condition is provably warp-uniform, so the code after a wait is not treated as divergent —
// otherwise every later shuffle is wrapped in a collective WARPSYNC loop)
__device__ __noinline__ void wait_ge_slow(const int* p, int v) {
  do {
    __nanosleep(64);
  } while (__any_sync(0xffffffffu, ld_acquire(p) < v));
}
__device__ __forceinline__ void wait_ge(const int* p, int v) {
  if (__any_sync(0xffffffffu, ld_acquire(p) < v)) wait_ge_slow(p, v);
}

// accumulator layout (lane 4 gid + q: row gid, columns 2q, 2q+1) -> m8n8k4 A fragments (A[gid][tig], A[gid][4+tig])
__device__ __forceinline__ void afrag(double x0, double x1, double& a0, double& a1, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const int s0 = 4 * gid + (tig >> 1);
  const double p0 = __shfl_sync(0xffffffffu, x0, s0), p1 = __shfl_sync(0xffffffffu, x1, s0);
  const double q0 = __shfl_sync(0xffffffffu, x0, s0 + 2), q1 = __shfl_sync(0xffffffffu, x1, s0 + 2);
  a0 = (tig & 1) ? p1 : p0;
  a1 = (tig & 1) ? q1 : q0;
}
// accumulator layout -> B fragments (B[tig][gid], B[4+tig][gid])
__device__ __forceinline__ void bfrag(double x0, double x1, double& b0, double& b1, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const int s0 = 4 * tig + (gid >> 1);
  const double p0 = __shfl_sync(0xffffffffu, x0, s0), p1 = __shfl_sync(0xffffffffu, x1, s0);
  const double q0 = __shfl_sync(0xffffffffu, x0, s0 + 16), q1 = __shfl_sync(0xffffffffu, x1, s0 + 16);
  b0 = (gid & 1) ? p1 : p0;
  b1 = (gid & 1) ? q1 : q0;
}
// store an accumulator-layout 8x8 tile in B-fragment order: element (r, c) at (r >> 2) 32 + 4 c + (r & 3), so a
// later B-fragment load is T[lane] (k-step 0) and T[32 + lane] (k-step 1): 256 contiguous bytes per warp
__device__ __forceinline__ void st_bfrag(double* T, double v0, double v1, int lane) {
  const int gid = lane >> 2, q = lane & 3;
  const int o = (gid >> 2) * 32 + 8 * q + (gid & 3);
  T[o] = v0;
  T[o + 4] = v1;
}
__device__ __forceinline__ double lds_v(const double* p) {   // ordered shared load (keeps register pressure low)
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(smem_u32(p)));
  return v;
}

// 8x8 LU in registers, natural order with the GEPP check (DESIGN R16): (x0, x1) hold the block in the
// accumulator layout (lane 4r + q: entries (r, 2q), (r, 2q+1)) and become L\U; L^-1 goes to linv (row-major,
// stride kLdL), U^-1 to uinv in B-fragment order. The elimination broadcasts per step the pivot, this lane's
// pivot-column entry and the pivot row at its two columns (4 shuffles); the inverses follow by column-parallel
// substitution from a shared-memory copy (lanes 0-7: columns of L^-1; lanes 8-15: columns of U^-1 through the
// reversal J U J), with the pivot reciprocals kept. Returns whether any check failed (warp-uniform).
__device__ __forceinline__ bool lu8_reg(double& x0, double& x1, double* stage, double* linv, double* uinv, int lane) {
  const int r = lane >> 2, q = lane & 3;
  const int j0 = 2 * q, j1 = 2 * q + 1;
  bool viol = false;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double v = (c & 1) ? x1 : x0;
    const double piv = __shfl_sync(0xffffffffu, v, 4 * c + (c >> 1));
    const double arc = __shfl_sync(0xffffffffu, v, 4 * r + (c >> 1));
    const double u0 = __shfl_sync(0xffffffffu, x0, 4 * c + q);
    const double u1 = __shfl_sync(0xffffffffu, x1, 4 * c + q);
    const double rp = rcp_fast(piv);
    if (lane == 0) stage[64 + c] = rp;
    const double l = arc * rp;
    const bool lrow = r > c;
    viol |= lrow & (fabs(arc) > fabs(piv));
    viol |= (r == c) & pivot_bad(piv);
    const double n0 = fma(-l, u0, x0), n1 = fma(-l, u1, x1);
    x0 = (lrow & (j0 > c)) ? n0 : x0;
    x0 = (lrow & (j0 == c)) ? l : x0;
    x1 = (lrow & (j1 > c)) ? n1 : x1;
    x1 = (lrow & (j1 == c)) ? l : x1;
  }
  *reinterpret_cast<double2*>(stage + r * 8 + j0) = make_double2(x0, x1);
  __syncwarp();
  if (lane < 16) {
    const bool isU = lane >= 8;
    const int j = lane & 7;
    double y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) y[k] = k == j ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (isU) y[k] *= lds_v(stage + 64 + 7 - k);
#pragma unroll
      for (int i = k + 1; i < 8; ++i) y[i] = fma(-lds_v(stage + (isU ? (7 - i) * 8 + 7 - k : i * 8 + k)), y[k], y[i]);
    }
    if (!isU) {
#pragma unroll
      for (int i = 0; i < 8; ++i) linv[i * kLdL + j] = y[i];
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = 7 - i, cc = 7 - j;   // U^-1[rr][cc]
        uinv[(rr >> 2) * 32 + 4 * cc + (rr & 3)] = y[i];
      }
    }
  }
  __syncwarp();
  return __any_sync(0xffffffffu, viol);
}

// instrumentation (hdg_debug_set_trace): per task of CTA 0 (first 512 tasks), [warp, claim, k-loop done, wavefront
// ready, diagonal block done, end, sm clock at claim] as clock64 stamps
#define RW_STAMP(k)                                                                              \
  do {                                                                                           \
    if (a.trace && blockIdx.x == 0 && q < 512 && lane == 0) a.trace[(int64_t)q * 8 + (k)] = clock64(); \
  } while (0)

template <int NWARPS, int NCTM, int TAM>
__global__ void __launch_bounds__(NWARPS * 32, 1) rows_kernel(const CondenseArgs a, const RowCfg cfg) {
  extern __shared__ __align__(128) double smem[];
  const RowGeo G(a.ne, a.nf);
  const int ne = G.ne, nf = G.nf, RA = G.RA, TA = G.TA, nct = G.NCT, NT = G.NT;
  int* ctrl = reinterpret_cast<int*>(smem);
  int* next_task = ctrl;
  int* fin = ctrl + 1;          // [4] tasks finished per slot (monotonic)
  int* prog = ctrl + 8;         // [4][32] per slot and A row tile: t * 64 + U tiles published (monotonic)
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int gid = lane >> 2, tig = lane & 3;
  double* stage = smem + kCtrlInts / 2 + warp * kWScr;
  double* linv = stage + 72;
  double* nxt = stage + 168;    // the k loop's hand-over tile (8 x 8, row stride kLdL)
  double* pool = smem + kCtrlInts / 2 + NWARPS * kWScr;
  for (int i = threadIdx.x; i < kCtrlInts; i += blockDim.x) ctrl[i] = 0;
  __syncthreads();

  const int n_local = (int)((a.count - blockIdx.x + gridDim.x - 1) / gridDim.x);
  const int total = n_local * NT;
  // U tile (k, j) of slot s
  auto urow = [&](int s, int k) -> double* {
    if (cfg.overlap) return pool + (s == 0 ? G.row_off(k) : cfg.P - G.row_off(k + 1));
    return pool + (int64_t)s * G.tiles * 64 + G.row_off(k);
  };

#pragma unroll 1
  for (;;) {
    int q = 0;
    if (lane == 0) q = atomicAdd(next_task, 1);
    q = __shfl_sync(0xffffffffu, q, 0);
    if (q >= total) break;
    RW_STAMP(1);
    if (a.trace && blockIdx.x == 0 && q < 512 && lane == 0) a.trace[(int64_t)q * 8] = warp;
    // task order (every wait points at an earlier task: the lowest unfinished task never waits). An element's C
    // row tiles wait for its whole chain of diagonal blocks, so they are placed one element later, after the next
    // element's head rows (whose chain then starts while this one's C rows are still pending):
    //   A(0) | H(1) C(0) T(1) | H(2) C(1) T(2) | ... | C(n-1)
    // H = A row tiles [0, hr), T = [hr, TA): the rows of an overlapping slot that wait for the previous element
    // (hr = cfg.ovl in overlap mode, else TA).
    // Disjoint slots (NS >= 2): the C rows are delayed by D = NS - 1 elements, so up to NS elements' chains are
    // in flight:  A(0) .. A(D-1) | A(D) C(0) | A(D+1) C(1) | ... | C(n-D) .. C(n-1)
    // (A(p+D) reuses the slot of element p+D-NS < p, whose C rows come earlier).
    int t, tile;
    {
      const int TC = NT - TA;
      if (cfg.overlap) {
        const int hr = cfg.ovl;
        if (q < TA) {
          t = 0;
          tile = q;
        } else {
          const int qq = q - TA, p = qq / NT, r = qq - p * NT;
          if (p >= n_local - 1) { t = p; tile = TA + r; }              // the last element's C rows
          else if (r < hr) { t = p + 1; tile = r; }                     // H(p+1)
          else if (r < hr + TC) { t = p; tile = TA + (r - hr); }        // C(p)
          else { t = p + 1; tile = r - TC; }                            // T(p+1)
        }
      } else {
        const int D = min(cfg.D, n_local), Pm = n_local - D;
        if (q < D * TA) {
          t = q / TA;
          tile = q - t * TA;
        } else if (q - D * TA < Pm * NT) {
          const int qq = q - D * TA, p = qq / NT, r = qq - p * NT;
          if (r < TA) { t = p + D; tile = r; }
          else { t = p; tile = r; }
        } else {
          const int qq = q - D * TA - Pm * NT;
          t = Pm + qq / TC;
          tile = TA + qq % TC;
        }
      }
    }
    const int s = t % cfg.NS;
    if (a.trace && blockIdx.x == 0 && q < 512 && lane == 0) {
      a.trace[(int64_t)q * 8 + 6] = t;
      a.trace[(int64_t)q * 8 + 7] = tile;
    }
    const int64_t it = blockIdx.x + (int64_t)t * gridDim.x;
    const int64_t l = a.elems ? a.elems[it] : it;
    const bool isA = tile < TA;
    const int i = isA ? tile : tile - TA;   // A row tile, or C row tile
    int* prog_s = prog + s * 32;
    const int tb = t * 64;
    double* LU = reinterpret_cast<double*>(a.factors + a.offF[l]);

    if (isA && tile == 0) {
      if (lane == 0 && it + gridDim.x < a.count) {   // the CTA's next element into L2
        const int64_t ln = a.elems ? a.elems[it + gridDim.x] : it + gridDim.x;
        prefetch_l2(a.A + a.offA[ln], (uint32_t)(ne * ne * 8));
        prefetch_l2(a.B + a.offB[ln], (uint32_t)(ne * nf * 8));
        prefetch_l2(a.C + a.offC[ln], (uint32_t)(nf * ne * 8));
        prefetch_l2(a.D + a.offD[ln], (uint32_t)(nf * nf * 8));
      }
      int32_t* perm = reinterpret_cast<int32_t*>(LU + (int64_t)ne * ne);
      for (int r = lane; r < ne; r += 32) perm[r] = r;
    }

    // ---- the row tile into registers (accumulator layout; identity padding rows of A, zero padding elsewhere).
    //      Branch-free: every load of the tile is issued before any is used (one memory latency per task).
    double x[NCTM][2];
    {
      const int r = 8 * i + gid;
      const bool real = isA ? r < ne : r < nf;
      const int rr = real ? r : 0;
      const double* P0 = isA ? a.A + a.offA[l] + (int64_t)rr * ne : a.C + a.offC[l] + (int64_t)rr * ne;
      const double* P1 = isA ? a.B + a.offB[l] + (int64_t)rr * nf : a.D + a.offD[l] + (int64_t)rr * nf;
      const double vlast = real ? __ldg(isA ? a.re + a.offRe[l] + r : a.rf + a.offRf[l] + r) : 0.0;
      const double shv = (isA && real && a.shift) ? __ldg(a.shift + a.offRe[l] + r) : 0.0;
#pragma unroll
      for (int j = 0; j < NCTM; ++j) {
        const int c0 = 8 * j + 2 * tig;
        const bool in0 = c0 < ne, in1 = c0 >= RA && c0 - RA < nf;
        const double* p = in0 ? P0 + c0 : P1 + (c0 - RA);
        double2 v = make_double2(0.0, 0.0);
        if (real && j < nct && (in0 || in1)) v = __ldg(reinterpret_cast<const double2*>(p));
        x[j][0] = v.x;
        x[j][1] = v.y;
      }
#pragma unroll
      for (int j = 0; j < NCTM; ++j) {
        const int c0 = 8 * j + 2 * tig;
        if (real && c0 - RA == nf) x[j][0] = vlast;                       // the r_e / r_f column
        if (j == i) {                                                     // re-condensation: A_e + diag(shift_e)
          if (c0 == r) x[j][0] += shv;                                    // (the diagonal is in tile i)
          if (c0 + 1 == r) x[j][1] += shv;
        }
        if (isA && !real) {                                               // identity padding rows of A
          x[j][0] = c0 == r ? 1.0 : 0.0;
          x[j][1] = c0 + 1 == r ? 1.0 : 0.0;
        }
      }
    }
    const int rowg = 8 * i + gid;             // this lane's row (A rows: of A_e; C rows: of C_e)
    const bool rreal = isA ? rowg < ne : rowg < nf;
    bool viol = false;

    // ---- the k loop (a runtime loop: one compact copy of the code — the instruction cache holds it): for each
    //      row tile k < kend, L_ik = M_ik U_kk^-1 (A rows: the GEPP multipliers, checked; kept in x[k] for the
    //      factor record) and M_i,>k -= L_ik U_k,>k. M_ik reaches the loop through the per-warp tile `nxt` (stored
    //      by the previous iteration's update of column tile k), so no register of x is indexed at run time.
    //      For an A row tile the last k (= i-1) is the wavefront: only the diagonal block's update here, the rest
    //      interleaved with this row's own TRSM below.
    const int kend = isA ? i : TA;
    double2 nlast = make_double2(0.0, 0.0);    // -L_{i,i-1} as A fragments (the wavefront update)
    if (kend > 0) *reinterpret_cast<double2*>(nxt + gid * kLdL + 2 * tig) = make_double2(x[0][0], x[0][1]);
#pragma unroll 1
    for (int k = 0; k < kend; ++k) {
      const bool wave = isA && k == i - 1;
      const double* Uk = urow(s, k);
      __syncwarp();
      const double a0 = nxt[gid * kLdL + tig], a1 = nxt[gid * kLdL + 4 + tig];
      wait_ge(prog_s + k, tb + (wave ? 2 : nct - k));   // the wavefront needs U_kk^-1 and the tile (k, i) first
      // (chunked waits on every k — consuming U rows as they are published — measured slower: C4 82 vs 66 ms)
      double L[2] = {0.0, 0.0};
      dmma(L, a0, Uk[lane]);
      dmma(L, a1, Uk[32 + lane]);
      if (isA) viol |= fabs(L[0]) > 1.0 || fabs(L[1]) > 1.0;
      double n0, n1;
      afrag(L[0], L[1], n0, n1, lane);
      n0 = -n0;
      n1 = -n1;
      __syncwarp();
#pragma unroll
      for (int j = 0; j < NCTM; ++j) {
        if (j == k) {   // L_ik (A rows: stored with the row at the end of the task)
          x[j][0] = L[0];
          x[j][1] = L[1];
        }
        if (j > k && j < nct && (!wave || j == k + 1)) {
          const double* T = Uk + 64 * (j - k);
          dmma(x[j], n0, T[lane]);
          dmma(x[j], n1, T[32 + lane]);
          if (j == k + 1) *reinterpret_cast<double2*>(nxt + gid * kLdL + 2 * tig) = make_double2(x[j][0], x[j][1]);
        }
      }
      if (wave) nlast = make_double2(n0, n1);
    }
    RW_STAMP(2);

    if (isA) {
      // this slot's U rows are reused: the element that used them before must be complete (and, where the two
      // slots overlap, the previous element too)
      if (t >= cfg.NS) wait_ge(fin + s, (t / cfg.NS) * NT);
      if (cfg.overlap && i >= cfg.ovl && t >= 1) wait_ge(fin + (s ^ 1), ((t - 1) / 2 + 1) * NT);
      RW_STAMP(3);
      // ---- the diagonal block: L_ii U_ii with both inverses; U_ii^-1 published at once
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int j = 0; j < TAM; ++j)
        if (j == i) { d0 = x[j][0]; d1 = x[j][1]; }
      double* Ui = urow(s, i);
      viol |= lu8_reg(d0, d1, stage, linv, Ui, lane);
#pragma unroll
      for (int j = 0; j < TAM; ++j)
        if (j == i) { x[j][0] = d0; x[j][1] = d1; }
      __syncwarp();
      if (lane == 0) st_release(prog_s + i, tb + 1);
      RW_STAMP(4);
      // ---- U_i,>i = L_ii^-1 M_i,>i tile by tile, each tile first receiving the wavefront update from row i-1.
      //      Publication points (ready = tiles of row i from its diagonal): after tiles i+1 and i+2 (the next row
      //      tile's diagonal update and its first TRSM tile), then every kGrp tiles, and the last; the consumer
      //      waits at the matching points.
      const double la0 = linv[gid * kLdL + tig], la1 = linv[gid * kLdL + 4 + tig];
      const int k = i - 1;
      const double* Uk = urow(s, k >= 0 ? k : 0);
      // the L part and the diagonal block go to the factor record now; the columns right of the diagonal are
      // handed to the (runtime) TRSM loop through their own U-store tiles, in B-fragment order
      if (rreal) {
#pragma unroll
        for (int j = 0; j < TAM; ++j)
          if (j <= i && 8 * j + 2 * tig < ne)
            *reinterpret_cast<double2*>(LU + (int64_t)rowg * ne + 8 * j + 2 * tig) = make_double2(x[j][0], x[j][1]);
      }
#pragma unroll
      for (int j = 1; j < NCTM; ++j)
        if (j > i && j < nct) st_bfrag(Ui + 64 * (j - i), x[j][0], x[j][1], lane);
      const int ao = (gid >> 2) * 32 + 8 * tig + (gid & 3);   // this lane's accumulator pair in a B-order tile
      // groups of kGrp tiles (the first group 2: the next row tile's first needs), the tiles of a group
      // independent (their latencies overlap); one wait and one publication per group
#pragma unroll 1
      for (int j0 = i + 1; j0 < nct;) {
        const int gsz = j0 == i + 1 ? 2 : kGrp;
        const int jend = min(j0 + gsz, nct);
        if (i >= 1) wait_ge(prog_s + k, tb + jend - k);
        __syncwarp();
#pragma unroll
        for (int g = 0; g < kGrp; ++g) {
          const int j = j0 + g;
          if (j < jend) {
            double* T = Ui + 64 * (j - i);
            double acc[2] = {T[ao], T[ao + 4]};
            if (i >= 1) {
              const double* Tk = Uk + 64 * (j - k);
              dmma(acc, nlast.x, Tk[lane]);
              dmma(acc, nlast.y, Tk[32 + lane]);
            }
            double b0, b1;
            bfrag(acc[0], acc[1], b0, b1, lane);
            double u[2] = {0.0, 0.0};
            dmma(u, la0, b0);
            dmma(u, la1, b1);
            T[ao] = u[0];
            T[ao + 4] = u[1];
          }
        }
        __syncwarp();
        if (lane == 0) st_release(prog_s + i, tb + (jend - i));
        j0 = jend;
      }
      // the U part of the factor record's row tile, read back from the published tiles (after every publication:
      // a release orders all earlier memory operations, the global stores must not sit in front of one)
      __syncwarp();
      if (rreal) {
#pragma unroll 1
        for (int j = i + 1; j < TA; ++j)
          if (8 * j + 2 * tig < ne) {
            const double* T = Ui + 64 * (j - i);
            *reinterpret_cast<double2*>(LU + (int64_t)rowg * ne + 8 * j + 2 * tig) = make_double2(T[ao], T[ao + 4]);
          }
      }
    } else {
      // ---- C row tile: its [D | r_f] columns now hold [S_e | g_e]
      const SgDst dst = sg_dst(a, l);
#pragma unroll
      for (int j = 0; j < NCTM; ++j)
        if (j >= TA && j < nct && rreal) {
          const int c0 = 8 * (j - TA) + 2 * tig;
          if (c0 < nf) out_S2(dst, nf, rowg, c0, x[j][0], x[j][1]);
          else if (c0 == nf) out_g(dst, rowg, x[j][0]);
        }
    }

    // ---- task done: mark a failed speculation, count the task; the element's last task settles the element
    RW_STAMP(5);
    viol = __any_sync(0xffffffffu, viol);
    if (viol && lane == 0) a.mark[l] = 1;
    __syncwarp();
    if (lane == 0) {
      const int old = atom_add_acq_rel(fin + s, 1);
      if (old + 1 == (t / cfg.NS + 1) * NT) {
        if (a.mark[l]) {
          a.mark[l] = 0;
          a.redo[atomicAdd(a.redo_count, 1)] = (int32_t)l;
        } else {
          a.info[l] = 0;
        }
      }
    }
  }
}

template <int NWARPS, int NCTM, int TAM>
cudaError_t launch_rows_t(const CondenseArgs& a, const RowCfg& cfg, int64_t smem, int sms, cudaStream_t s) {
  auto kern = rows_kernel<NWARPS, NCTM, TAM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t grid = std::min<int64_t>(sms, a.count);
  grid = grid_cap(grid);
  kern<<<(unsigned)grid, NWARPS * 32, (size_t)smem, s>>>(a, cfg);
  return cudaGetLastError();
}

// warps per CTA (HDG_ROWS_WARPS=8|12 for experiments; default 12)
int rows_warps() {
  static const int w = [] {
    const char* v = getenv("HDG_ROWS_WARPS");
    return v && atoi(v) == 8 ? 8 : 12;
  }();
  return w;
}

bool rows_config(int ne, int nf, size_t smem_optin, RowCfg* cfg, int64_t* smem_bytes) {
  const RowGeo G(ne, nf);
  if (G.TA > 16 || G.NCT > 28) return false;
  const int64_t fixed = 8 * (kCtrlInts / 2 + (int64_t)rows_warps() * kWScr);
  const int64_t avail = ((int64_t)smem_optin - fixed) / 8 / 64 * 64;   // pool doubles, whole tiles
  const int64_t slot = G.tiles * 64;
  if (slot > avail) return false;
  RowCfg c{};
  if (2 * slot <= avail) {
    c.NS = (int)std::min<int64_t>(4, avail / slot);
    c.P = (int)(c.NS * slot);
    c.overlap = 0;
    c.ovl = G.TA;
    const char* dv = getenv("HDG_ROWS_DELAY");   // experiments: the C-row delay (1 .. NS - 1)
    c.D = dv ? std::max(1, std::min(c.NS - 1, atoi(dv))) : 1;   // (C3: D = 1 49.9, 2 49.8, 3 57.8 ms)
  } else {
    c.NS = 2;
    c.D = 1;
    c.P = (int)avail;
    c.overlap = 1;
    c.ovl = G.TA;
    for (int k = 0; k < G.TA; ++k)
      if (G.row_off(k + 1) > c.P - slot) { c.ovl = k; break; }
  }
  if (cfg) *cfg = c;
  if (smem_bytes) *smem_bytes = fixed + 8 * (int64_t)c.P;
  return true;
}

}  // namespace

bool rows_supported(int ne, int nf, size_t smem_optin) { return rows_config(ne, nf, smem_optin, nullptr, nullptr); }

cudaError_t launch_condense_rows(const CondenseArgs& a, int sms, size_t smem_optin, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  RowCfg cfg;
  int64_t smem = 0;
  if (!rows_config(a.ne, a.nf, smem_optin, &cfg, &smem)) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(a.redo_count, 0, sizeof(int32_t), s);
  if (e != cudaSuccess) return e;
  const RowGeo G(a.ne, a.nf);
  ++*launches;
  // (NCTM, TAM) = register column tiles and A row tiles, compile-time: C3 (16, 8), C4 (22 -> 24, 15 -> 16), C5's
  // n_e = 36 / 72 / 120 buckets
  const int nw = rows_warps();
  auto pick = [&](auto nwc) -> cudaError_t {
    constexpr int NW = decltype(nwc)::value;
    if (G.TA <= 8 && G.NCT <= 16) return launch_rows_t<NW, 16, 8>(a, cfg, smem, sms, s);
    if (G.TA <= 12 && G.NCT <= 20) return launch_rows_t<NW, 20, 12>(a, cfg, smem, sms, s);
    if (G.TA <= 16 && G.NCT <= 24) return launch_rows_t<NW, 24, 16>(a, cfg, smem, sms, s);
    return launch_rows_t<NW, 28, 16>(a, cfg, smem, sms, s);
  };
  e = nw == 8 ? pick(std::integral_constant<int, 8>{}) : pick(std::integral_constant<int, 12>{});
  if (e != cudaSuccess) return e;
  // the elements whose speculation failed, on the exact path (an empty list costs one short launch)
  ++*launches;
  return launch_exact_list(a, a.redo, a.redo_count, sms, s);
}

}  // namespace hdg
