// condense_sweep.cu — rows a1-a5 of the hot path for every (n_e, n_f) class whose working set
// fits one SM's shared memory: the "sweep" condensation kernel.
//
// For each element e (Eq. hybridsystem; "condense"):
//     S_e = D_e - C_e A_e^-1 B_e,   g_e = r_f - C_e A_e^-1 r_e,
// with A_e factored by Gaussian elimination with partial pivoting (GEPP); the factorization is
// kept for the reconstruction.
//
// Formulation. One right-looking blocked elimination sweep (panels of 16 columns of A_e) over
//     T = [A_e | B_e | r_e]   (n_e rows, shared memory)   and   Cr = C_e   (n_f rows, A columns only, shared memory)
// with P A_e = L U:  T <- [L\U | W = L^-1 P [B_e r_e]],  Cr <- Y = C_e U^-1,  and since
//     C_e A_e^-1 [B_e r_e] = (C_e U^-1)(L^-1 P [B_e r_e]) = Y W,
// the Schur complement [S_e | g_e] = [D_e | r_f] - sum_p Y_p W_p is accumulated panel by panel in REGISTERS
// (DMMA accumulator tiles owned by the worker warps, initialised from D_e / r_f), so there is neither a backward
// substitution phase nor a separate Schur GEMM at the end. Per panel p (columns jb..jb+16):
//   warp 0 (the chain warp): look-ahead — L21/U12 tiles of the next diagonal block, its update, and the
//       factorization of the next 16x16 diagonal block in registers (diag_chain: L\U, L^-1 and U^-1 in ONE
//       16-step loop, pivot row broadcast by shuffles);
//   warps 1.. (workers): TRSM tiles L21 = A21 U11^-1 (A rows), Y_p = C_p U11^-1 (C rows), U12 = L11^-1 A12 (all
//       columns right of the panel, incl. W), then the trailing updates of the A rows and C rows and the
//       register-resident [S|g] update -= Y_p W_p — all FP64 tensor-core MMAs (mma.sync m8n8k4, 16x32 blocks).
// Pivoting is speculative (R16): every multiplier of the natural-order elimination is checked; if any
// |l_ik| > 1 (GEPP would have interchanged rows) or a pivot is zero/subnormal, the whole CTA aborts the element
// (__syncthreads_or) and redoes it on the exact path: unblocked GEPP with the warp-level pivot search (maximal
// |a_ik|, lowest index on ties). When the check passes, GEPP's pivot sequence is the identity
// and the fast path IS GEPP.
// Data movement: TMA bulk copies (cp.async.bulk + mbarrier transaction counts) stage A_e rows, B_e rows and C_e
// rows; the L\U rows of each finished panel leave by TMA bulk stores (shared -> global) while the sweep goes on;
// the next element's blocks are prefetched into L2 at the start of the current one.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "dev_common.cuh"
#include "hdg_internal.cuh"

namespace hdg {
namespace {

constexpr int NB = kSweepNB;   // panel width (see diag_block for NB = 8 / 16)

// instrumentation (hdg_debug_set_trace): clock64 stamp k of element-iteration it, CTA 0, warps 0 and 1
#define SW_STAMP(it, k)                                                                                       \
  do {                                                                                                      \
    if (a.trace && blockIdx.x == 0 && (it) < 4 && (threadIdx.x == 0 || threadIdx.x == blockDim.x - 32))     \
      a.trace[(it) * 256 + (threadIdx.x == 0 ? 128 : 0) + (k)] = clock64();                                 \
  } while (0)
constexpr int LDI = 20;   // row stride of the 16x16 inverse buffers

constexpr int kHelperShare = 14;   // 64ths of a panel's trailing blocks taken by the helper warp (see the trailing loop)
constexpr int BCW = 36;   // doubles per spare chain-warp slot (two slots: the 8x8 LU's staging copy)

// ------------------------------------------------------------------------------------------------------------
// lu8: GEPP-checked natural-order LU of the 8x8 block at (r0, r0) of X (valid size nbv <= 8, identity padding),
// with L^-1 and U^-1 (8x8, row stride LDI) into Li8 / Ui8. Lane 4r + q holds entries (r, 2q) and (r, 2q + 1) — the
// m8n8 accumulator layout — so an elimination step broadcasts just the pivot, this lane's row entry in the pivot
// column and the pivot row at this lane's two columns (4 shuffles; the row-per-lane form needs 9 per step and
// measured 1.55 K vs 1.34 K cycles per call). The inverses follow by column-parallel forward substitution from a
// shared-memory copy of L\U (stage, 64 doubles): lanes 0-7 column j of L^-1, lanes 8-15 column j of U^-1 through
// the reversal J U J (lower triangular), with the pivot reciprocals kept from the elimination. Writes L\U rows
// < nbv back to X and to LU.
template <bool CS>
__device__ __forceinline__ bool lu8(double* X, int ld, int r0, int nbv, double* Li8, double* Ui8, double* LU, int ne,
                                    double* stage, int lane) {
  __syncwarp();
  const int r = lane >> 2, q = lane & 3;
  const int j0 = 2 * q, j1 = 2 * q + 1;
  double x0, x1;
  {
    const bool real = r < nbv;
    double2 v = make_double2(0.0, 0.0);
    if (real && j0 < nbv) v = *reinterpret_cast<const double2*>(X + (size_t)(r0 + r) * ld + r0 + j0);
    x0 = real ? (j0 < nbv ? v.x : 0.0) : (j0 == r ? 1.0 : 0.0);
    x1 = real ? (j1 < nbv ? v.y : 0.0) : (j1 == r ? 1.0 : 0.0);
  }
  bool viol = false;
  double rps[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double v = (c & 1) ? x1 : x0;
    const double piv = __shfl_sync(0xffffffffu, v, 4 * c + (c >> 1));
    const double arc = __shfl_sync(0xffffffffu, v, 4 * r + (c >> 1));
    const double u0 = __shfl_sync(0xffffffffu, x0, 4 * c + q);
    const double u1 = __shfl_sync(0xffffffffu, x1, 4 * c + q);
    const double rp = rcp_fast(piv);
    rps[c] = rp;
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
  if (r < nbv && j0 < nbv) {
    *reinterpret_cast<double2*>(X + (size_t)(r0 + r) * ld + r0 + j0) = make_double2(x0, x1);
    st_lu<CS>(LU + (size_t)(r0 + r) * ne + r0 + j0, x0, x1);
  }
  *reinterpret_cast<double2*>(stage + r * 8 + j0) = make_double2(x0, x1);
  __syncwarp();
  const bool isU = (lane & 8) != 0;
  const int j = lane & 7;
  double m[8][8], y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    y[k] = k == j ? 1.0 : 0.0;
#pragma unroll
    for (int i = k + 1; i < 8; ++i) m[i][k] = stage[isU ? (7 - i) * 8 + 7 - k : i * 8 + k];
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    y[k] = isU ? y[k] * rps[7 - k] : y[k];
#pragma unroll
    for (int i = k + 1; i < 8; ++i) y[i] = fma(-m[i][k], y[k], y[i]);
  }
  double* d0 = isU ? Ui8 + 7 * LDI + 7 - j : Li8 + j;
  const int rs = isU ? -LDI : LDI;
  if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 8; ++i) d0[i * rs] = y[i];
  }
  __syncwarp();
  return __any_sync(0xffffffffu, viol);
}

// acc (8x8, m8n8 accumulator layout) += sgn * P (8x8, row-major stride lp) * Q (8x8, row-major stride lq)
__device__ __forceinline__ void mm8(double (&acc)[2], const double* P, int lp, const double* Q, int lq, double sgn,
                                    int lane) {
  const int gid = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int k = 0; k < 8; k += 4) dmma(acc, sgn * P[gid * lp + k + tig], Q[(k + tig) * lq + gid]);
}
__device__ __forceinline__ void st8(double* D, int ld, const double (&acc)[2], int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  *reinterpret_cast<double2*>(D + gid * ld + 2 * tig) = make_double2(acc[0], acc[1]);
}

// diag_chain: the 16x16 diagonal block at (jb, jb) of T (valid size nb <= 16) factored as two 8x8 LUs:
//   L1 U1 = D11;  L21 = D21 U1^-1,  U12 = L1^-1 D12  (DMMA);  L2 U2 = D22 - L21 U12;
// and the 16x16 inverses assembled from the 8x8 ones, in place in Linv / Uinv (16 x LDI):
//   L^-1 = [[L1^-1, 0], [-L2^-1 (L21 L1^-1), L2^-1]],   U^-1 = [[U1^-1, -U1^-1 (U12 U2^-1)], [0, U2^-1]].
// Same pivot order and GEPP check as a 16-step elimination (every multiplier |l| <= 1, pivots normal), with
// half the broadcast traffic per step and a quarter of the code (measured on the box: the fully unrolled 16-step
// body spends ~2x its standalone time in the kernel, instruction fetch). L\U goes to T and the factor record LU.
template <bool CS>
__device__ __forceinline__ bool diag_chain(double* T, int ldT, int jb, int nb, double* Linv, double* Uinv,
                                           double* stage, double* LU, int ne, int lane) {
  __syncwarp();
  const int n1 = nb < 8 ? nb : 8, n2 = nb > 8 ? nb - 8 : 0;
  bool viol = lu8<CS>(T, ldT, jb, n1, Linv, Uinv, LU, ne, stage, lane);
  const int gid = lane >> 2, tig = lane & 3, c = 2 * tig;
  double* D12 = T + (size_t)jb * ldT + jb + 8;
  double* D21 = T + (size_t)(jb + 8) * ldT + jb;
  double* D22 = D21 + 8;
  if (n2 > 0) {
    // L21 = D21 U1^-1 (multipliers: GEPP check), U12 = L1^-1 D12
    double l21[2] = {0.0, 0.0}, u12[2] = {0.0, 0.0};
    mm8(l21, D21, ldT, Uinv, LDI, 1.0, lane);
    mm8(u12, Linv, LDI, D12, ldT, 1.0, lane);
    __syncwarp();
    if (gid < n2) {
      viol |= fabs(l21[0]) > 1.0 || fabs(l21[1]) > 1.0;
      st8(D21, ldT, l21, lane);
      st_lu<CS>(LU + (size_t)(jb + 8 + gid) * ne + jb + c, l21[0], l21[1]);
    }
    if (c < n2) {
      *reinterpret_cast<double2*>(D12 + gid * ldT + c) = make_double2(u12[0], u12[1]);
      st_lu<CS>(LU + (size_t)(jb + gid) * ne + jb + 8 + c, u12[0], u12[1]);
    }
    __syncwarp();
    // D22 -= L21 U12 (entries of D22 outside the valid block are neither read nor written)
    double d22[2];
    d22[0] = (gid < n2 && c < n2) ? D22[gid * ldT + c] : 0.0;
    d22[1] = (gid < n2 && c + 1 < n2) ? D22[gid * ldT + c + 1] : 0.0;
    mm8(d22, D21, ldT, D12, ldT, -1.0, lane);
    __syncwarp();
    if (gid < n2 && c < n2) *reinterpret_cast<double2*>(D22 + gid * ldT + c) = make_double2(d22[0], d22[1]);
    __syncwarp();
  }
  viol |= lu8<CS>(T, ldT, jb + 8, n2, Linv + 8 * LDI + 8, Uinv + 8 * LDI + 8, LU, ne, stage, lane);
  // off-diagonal tiles of the inverses: stage P = L21 L1^-1 and Q = U12 U2^-1 in their final tiles, then
  // X = -L2^-1 P, Y = -U1^-1 Q; zero the other off-diagonal tiles
  double P[2] = {0.0, 0.0}, Q[2] = {0.0, 0.0};
  if (n2 > 0) {
    mm8(P, D21, ldT, Linv, LDI, 1.0, lane);
    mm8(Q, D12, ldT, Uinv + 8 * LDI + 8, LDI, 1.0, lane);
  }
  st8(Linv + 8 * LDI, LDI, P, lane);
  st8(Uinv + 8, LDI, Q, lane);
  *reinterpret_cast<double2*>(Linv + gid * LDI + 8 + c) = make_double2(0.0, 0.0);
  *reinterpret_cast<double2*>(Uinv + (8 + gid) * LDI + c) = make_double2(0.0, 0.0);
  __syncwarp();
  double X[2] = {0.0, 0.0}, Y[2] = {0.0, 0.0};
  mm8(X, Linv + 8 * LDI + 8, LDI, Linv + 8 * LDI, LDI, -1.0, lane);
  mm8(Y, Uinv, LDI, Uinv + 8, LDI, -1.0, lane);
  __syncwarp();
  st8(Linv + 8 * LDI, LDI, X, lane);
  st8(Uinv + 8, LDI, Y, lane);
  __syncwarp();
  return __any_sync(0xffffffffu, viol);
}

// The diagonal block of one panel: NB = 8 -> one 8x8 LU (its L^-1, U^-1 written straight into the Linv / Uinv
// buffers); NB = 16 -> the two-LU form above.
template <bool CS>
__device__ __forceinline__ bool diag_block(double* T, int ldT, int jb, int nb, double* Linv, double* Uinv,
                                           double* scratch, double* LU, int ne, int lane) {
  if constexpr (NB == 8) {
    __syncwarp();
    return lu8<CS>(T, ldT, jb, nb, Linv, Uinv, LU, ne, scratch, lane);
  } else {
    return diag_chain<CS>(T, ldT, jb, nb, Linv, Uinv, scratch, LU, ne, lane);
  }
}

// ------------------------------------------------------------------------------------------------------------
// prep_next (chain warp): the L21 rows [jn, r_hi) and U12 columns [jn, jn + nn8) of the NEXT diagonal block from
// panel (jb, nb), all 8 accumulator chains interleaved, stored to T (and the factor record), then that block's
// update D_{p+1} -= L21 U12. Returns whether a multiplier |l| > 1 appeared.
template <bool CS>
__device__ __forceinline__ bool prep_next(double* T, int ldT, int jb, int nb, int jn, int r_hi, int nn8,
                                          const double* Linv, const double* Uinv, double* LU, int ne, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const int nk4 = (nb + 3) >> 2, nb8t = (nb + 7) >> 3;
  const int nrtL = (r_hi - jn) >> 3, nctU = nn8 >> 3;
  double aL[2][4], bU[4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      aL[i][kk] = (i < nrtL && kk < nk4) ? T[(size_t)(jn + 8 * i + gid) * ldT + jb + 4 * kk + tig] : 0.0;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      bU[kk][j] = (j < nctU && kk < nk4) ? T[(size_t)(jb + 4 * kk + tig) * ldT + jn + 8 * j + gid] : 0.0;
  double accL[2][2][2], accU[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) accL[i][j][0] = accL[i][j][1] = accU[i][j][0] = accU[i][j][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    if (kk < nk4) {
      double ui[2], li[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) ui[j] = Uinv[(4 * kk + tig) * LDI + 8 * j + gid];
#pragma unroll
      for (int i = 0; i < 2; ++i) li[i] = Linv[(8 * i + gid) * LDI + 4 * kk + tig];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (i < nrtL && j < nb8t) dmma(accL[i][j], aL[i][kk], ui[j]);
          if (i < nb8t && j < nctU) dmma(accU[i][j], li[i], bU[kk][j]);
        }
    }
  }
  bool viol = false;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c = 8 * j + 2 * tig;
      if (i < nrtL && j < nb8t) {
        const int row = jn + 8 * i + gid;
        *reinterpret_cast<double2*>(T + (size_t)row * ldT + jb + c) = make_double2(accL[i][j][0], accL[i][j][1]);
        if (row < ne && c < nb) {
          viol |= fabs(accL[i][j][0]) > 1.0 || fabs(accL[i][j][1]) > 1.0;
          st_lu<CS>(LU + (size_t)row * ne + jb + c, accL[i][j][0], accL[i][j][1]);
        }
      }
      if (i < nb8t && j < nctU) {
        const int row = jb + 8 * i + gid, col = jn + c;
        *reinterpret_cast<double2*>(T + (size_t)row * ldT + col) = make_double2(accU[i][j][0], accU[i][j][1]);
        if (8 * i + gid < nb && col < ne)
          st_lu<CS>(LU + (size_t)row * ne + col, accU[i][j][0], accU[i][j][1]);
      }
    }
  __syncwarp();
  return viol;
}

// Row order of the accumulator tiles (and of their A operands) in the shared-memory updates: lane (gid, tig) of a
// DMMA m8n8k4 holds accumulator row gid; if that row is T row gid, a 16-byte accumulator access (quarter warp =
// rows gid, gid + 1) puts both rows in the same 64-byte half of the bank space for the row strides pad_ld picks
// (4 or 12 mod 16 doubles, which keep the 8-byte fragment loads conflict-free) — 2-way conflicts on every
// accumulator load and store (ncu: 30 % of the sweep kernel's shared wavefronts were conflict excess). Mapping
// accumulator row g to T row srow(g) = g with bits 0 and 1 swapped (0, 2, 1, 3, 4, 6, 5, 7) makes the quarter-warp
// row pairs (0, 2), (1, 3), ... land in opposite halves while the A fragments' 4-row phases keep 4 distinct bank
// groups. The product is unchanged: A rows and accumulator rows are permuted together.
__device__ __forceinline__ int srow(int g) { return (g & 4) | ((g & 1) << 1) | ((g >> 1) & 1); }

// L21-type TRSM tile: rows r0..r0+8 of X (stride ld), columns jb..jb+nb: X <- X U11^-1. Returns whether any
// multiplier |l| > 1 in a real (row < check_rows) position.
// nrt (1 or 2) row tiles r0.. at once: 4 independent accumulator chains. When LU != nullptr the multipliers of
// real rows (< check_rows = ne) are also stored to the factor record.
template <bool CS>
__device__ __forceinline__ bool trsm_right(double* X, int ld, int r0, int nrt, int jb, int nb, const double* Uinv,
                                           int check_rows, double* LU, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const int sg = srow(gid);   // accumulator / A-operand row of this lane (bank-conflict-free row order)
  const int nk4 = (nb + 3) >> 2, nct = (nb + 7) >> 3;
  double a[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      a[i][kk] = (i < nrt && kk < nk4) ? X[(size_t)(r0 + 8 * i + sg) * ld + jb + 4 * kk + tig] : 0.0;
  double acc[2][2][2] = {};
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    if (kk < nk4) {
      const double u0 = Uinv[(4 * kk + tig) * LDI + gid], u1 = Uinv[(4 * kk + tig) * LDI + 8 + gid];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (i < nrt) {
          // U^-1 is upper triangular: output columns 0-7 take only k < 8 (the skipped terms are exact zeros)
          if (kk < 2) dmma(acc[i][0], a[i][kk], u0);
          if (nct > 1) dmma(acc[i][1], a[i][kk], u1);
        }
      }
    }
  }
  bool viol = false;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = r0 + 8 * i + sg;
    const bool chk = row < check_rows;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (i < nrt && j < nct) {
        const int c = 8 * j + 2 * tig;
        if (chk && c < nb) viol |= fabs(acc[i][j][0]) > 1.0;
        if (chk && c + 1 < nb) viol |= fabs(acc[i][j][1]) > 1.0;
        *reinterpret_cast<double2*>(X + (size_t)row * ld + jb + c) = make_double2(acc[i][j][0], acc[i][j][1]);
        if (LU && chk && c < nb)
          st_lu<CS>(LU + (size_t)row * check_rows + jb + c, acc[i][j][0], acc[i][j][1]);
      }
    }
  }
  return viol;
}

// U12-type TRSM tile: rows jb..jb+nb (rounded up to 8) of T, columns c0..c0+8: T <- L11^-1 T. Columns < ne are
// U entries and are also stored to the factor record LU (row stride ne).
template <bool CS>
__device__ __forceinline__ void trsm_left(double* T, int ld, int jb, int nb, const double* Linv, int c0, int nct,
                                          double* LU, int ne, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const int sg = srow(gid);   // accumulator / A-operand row of this lane (bank-conflict-free row order)
  const int nk4 = (nb + 3) >> 2, nrt = (nb + 7) >> 3;
  double b[4][2];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      b[kk][j] = (kk < nk4 && j < nct) ? T[(size_t)(jb + 4 * kk + tig) * ld + c0 + 8 * j + gid] : 0.0;
  double acc[2][2][2] = {};
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    if (kk < nk4) {
      const double l0 = Linv[sg * LDI + 4 * kk + tig], l1 = Linv[(8 + sg) * LDI + 4 * kk + tig];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (j < nct) {
          // L^-1 is lower triangular: output rows 0-7 take only k < 8 (the skipped terms are exact zeros)
          if (kk < 2) dmma(acc[0][j], l0, b[kk][j]);
          if (nrt > 1) dmma(acc[1][j], l1, b[kk][j]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (i < nrt && j < nct) {
        const int col = c0 + 8 * j + 2 * tig;
        *reinterpret_cast<double2*>(T + (size_t)(jb + 8 * i + sg) * ld + col) = make_double2(acc[i][j][0], acc[i][j][1]);
        if (col < ne && 8 * i + sg < nb)
          st_lu<CS>(LU + (size_t)(jb + 8 * i + sg) * ne + col, acc[i][j][0], acc[i][j][1]);
      }
}

// Rank-nk update of one block: dst[r0 .. r0 + 8 nrt, c0 .. c0 + 8 nct) -= Ap[rows, 0..nk) * Bp[0..nk, cols).
// Ap/dst share row indices (strides lda/ldd), Bp/dst share column indices (stride ldb). nrt <= 2, nct <= 4.
__device__ __forceinline__ void upd_block(double* dst, int ldd, const double* Ap, int lda, const double* Bp, int ldb,
                                          int r0, int nrt, int c0, int nct, int nk, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const int sg = srow(gid);   // accumulator / A-operand row of this lane (bank-conflict-free row order)
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc[i][j][0] = 0.0;
      acc[i][j][1] = 0.0;
      if (i < nrt && j < nct) {
        const double2 v = *reinterpret_cast<const double2*>(dst + (size_t)(r0 + 8 * i + sg) * ldd + c0 + 8 * j + 2 * tig);
        acc[i][j][0] = v.x;
        acc[i][j][1] = v.y;
      }
    }
#pragma unroll
  for (int k = 0; k < NB; k += 4) {
    if (k < nk) {
      const double a0 = -Ap[(size_t)(r0 + sg) * lda + k + tig];
      const double a1 = nrt > 1 ? -Ap[(size_t)(r0 + 8 + sg) * lda + k + tig] : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j < nct) {
          const double b = Bp[(size_t)(k + tig) * ldb + c0 + 8 * j + gid];
          dmma(acc[0][j], a0, b);
          if (nrt > 1) dmma(acc[1][j], a1, b);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (i < nrt && j < nct)
        *reinterpret_cast<double2*>(dst + (size_t)(r0 + 8 * i + sg) * ldd + c0 + 8 * j + 2 * tig) =
            make_double2(acc[i][j][0], acc[i][j][1]);
}

// Full 16x32 block, k = 16: every fragment (2 x 4 A, 4 x 4 B) is loaded before the first MMA, so the 24 shared
// loads issue back to back and the 32 MMAs (8 independent accumulator chains) follow without load stalls.
__device__ __forceinline__ void upd_full16(double* dst, int ldd, const double* Ap, int lda, const double* Bp, int ldb,
                                           int r0, int c0, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const int sg = srow(gid);   // accumulator / A-operand row of this lane (bank-conflict-free row order)
  double a[4][2], b[4][4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    a[kk][0] = -Ap[(size_t)(r0 + sg) * lda + 4 * kk + tig];
    a[kk][1] = -Ap[(size_t)(r0 + 8 + sg) * lda + 4 * kk + tig];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[kk][j] = Bp[(size_t)(4 * kk + tig) * ldb + c0 + 8 * j + gid];
  }
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double2 v = *reinterpret_cast<const double2*>(dst + (size_t)(r0 + 8 * i + sg) * ldd + c0 + 8 * j + 2 * tig);
      acc[i][j][0] = v.x;
      acc[i][j][1] = v.y;
    }
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      dmma(acc[0][j], a[kk][0], b[kk][j]);
      dmma(acc[1][j], a[kk][1], b[kk][j]);
    }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<double2*>(dst + (size_t)(r0 + 8 * i + sg) * ldd + c0 + 8 * j + 2 * tig) =
          make_double2(acc[i][j][0], acc[i][j][1]);
}

// A rectangular trailing region [r_lo, r_hi) x [c_lo, c_hi) cut into 16x32 blocks (row remainder 8, column
// remainder 8/16/24); block index -> geometry.
struct Region {
  int r_lo, r_hi, c_lo, c_hi, nbc, nblk;
  __device__ Region(int rl, int rh, int cl, int ch) : r_lo(rl), r_hi(rh), c_lo(cl), c_hi(ch) {
    const int nbr = rh > rl ? (rh - rl + 15) >> 4 : 0;
    nbc = ch > cl ? (ch - cl + 31) >> 5 : 0;
    nblk = nbr * nbc;
  }
};

// ------------------------------------------------------------------------------------------------------------
// exact path: unblocked GEPP over [T | Cr] by the whole CTA (taken only when the speculation fails)
template <int THREADS>
__device__ void sweep_pivot(double* T, double* Cr, const SweepGeo& G, const double* A, const double* Bm,
                            const double* re, const double* Cm, const double* sh, int* piv, int* shared_fail, int tid) {
  const int ne = G.ne, nf = G.nf, ldT = G.ldT, ldC = G.ldC, CB = G.CB, NC = G.NCAB;
  // restage from global (zero padding everywhere); sh: the diagonal shift (re-condensation), NULL = none
  for (int i = tid; i < G.RA * ldT; i += THREADS) {
    const int row = i / ldT, col = i - row * ldT;
    double v = 0.0;
    if (row < ne) {
      if (col < ne) v = A[(size_t)row * ne + col] + ((sh && col == row) ? sh[row] : 0.0);
      else if (col >= CB && col < CB + nf) v = Bm[(size_t)row * nf + col - CB];
      else if (col == CB + nf) v = re[row];
    }
    T[i] = v;
  }
  for (int i = tid; i < G.NF8 * ldC; i += THREADS) {
    const int row = i / ldC, col = i - row * ldC;
    Cr[i] = (row < nf && col < ne) ? Cm[(size_t)row * ne + col] : 0.0;
  }
  if (tid == 0) *shared_fail = 0;
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  for (int k = 0; k < ne; ++k) {
    if (warp == 0) {
      double best = -1.0;
      int bi = 0x7fffffff;
      for (int r = k + lane; r < ne; r += 32) {
        const double v = fabs(T[(size_t)r * ldT + k]);
        if (v > best) { best = v; bi = r; }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) {
        const int pr = bi < ne ? bi : k;
        piv[k] = pr;
        const double pv = T[(size_t)pr * ldT + k];
        if (pv == 0.0 || pv != pv) *shared_fail = k + 1;   // zero or NaN pivot (DESIGN R7)
      }
    }
    __syncthreads();
    if (*shared_fail) break;
    const int pr = piv[k];
    if (pr != k)
      for (int j = tid; j < NC; j += THREADS) {
        const double t = T[(size_t)k * ldT + j];
        T[(size_t)k * ldT + j] = T[(size_t)pr * ldT + j];
        T[(size_t)pr * ldT + j] = t;
      }
    __syncthreads();
    const double pv = T[(size_t)k * ldT + k];
    // multipliers (a true division each, as the oracle) — A rows below k, then all C rows
    for (int i = k + 1 + tid; i < ne + nf; i += THREADS) {
      double* row = i < ne ? T + (size_t)i * ldT : Cr + (size_t)(i - ne) * ldC;
      row[k] = row[k] / pv;
    }
    __syncthreads();
    // rank-1 update: A rows over all columns > k, C rows over A columns > k
    const int wA = NC - k - 1, wC = ne - k - 1;
    const int nA = (ne - k - 1) * wA, nCw = nf * wC;
    for (int idx = tid; idx < nA + nCw; idx += THREADS) {
      if (idx < nA) {
        const int i = k + 1 + idx / wA, j = k + 1 + idx % wA;
        T[(size_t)i * ldT + j] = fma(-T[(size_t)i * ldT + k], T[(size_t)k * ldT + j], T[(size_t)i * ldT + j]);
      } else {
        const int q = idx - nA;
        const int i = q / wC, j = k + 1 + q % wC;
        Cr[(size_t)i * ldC + j] = fma(-Cr[(size_t)i * ldC + k], T[(size_t)k * ldT + j], Cr[(size_t)i * ldC + j]);
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------------------------
// The exact path of one element (all threads of the CTA), entirely in this CTA's global scratch slab X (so the
// TMA loads of the next element that are already in flight into shared memory are left alone). Not inlined:
// both roles call it.
template <int THREADS>
__device__ __noinline__ void exact_element(double* S_, double* g_, double* Kf, double* Ef, const int64_t* eblk,
                                           const int64_t* eE, const int32_t* so, const double* A, const double* Bm,
                                           const double* re, const double* Cm, const double* D, const double* rf,
                                           const double* sh, double* LU, int32_t* info, int ne, int nf, double* X,
                                           int* piv, int* sfail, int tid) {
  SgDst dst;
  dst.S = S_; dst.g = g_; dst.Kf = Kf; dst.Ef = Ef; dst.eblk = eblk; dst.eE = eE; dst.so = so;
  const SweepGeo G(ne, nf);
  const int ldT = G.ldT, ldC = G.ldC, CB = G.CB;
  double* T = X;
  double* Cr = X + (size_t)G.RA * ldT;
  __syncthreads();
  sweep_pivot<THREADS>(T, Cr, G, A, Bm, re, Cm, sh, piv, sfail, tid);
  const int fail = *sfail;
  if (fail) {
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    for (int i = tid; i < nf * nf; i += THREADS) out_S1(dst, nf, i / nf, i % nf, nan);
    for (int i = tid; i < nf; i += THREADS) out_g(dst, i, nan);
  } else {
    // [S | g] = [D | r_f] - Y W, ascending k
    for (int idx = tid; idx < nf * (nf + 1); idx += THREADS) {
      const int i = idx / (nf + 1), j = idx - i * (nf + 1);
      double sum = j < nf ? D[(size_t)i * nf + j] : rf[i];
      for (int k = 0; k < ne; ++k) sum = fma(-Cr[(size_t)i * ldC + k], T[(size_t)k * ldT + CB + j], sum);
      if (j < nf) out_S1(dst, nf, i, j, sum);
      else out_g(dst, i, sum);
    }
  }
  for (int idx = tid; idx < ne * ne; idx += THREADS) LU[idx] = T[(size_t)(idx / ne) * ldT + idx % ne];
  int32_t* perm = reinterpret_cast<int32_t*>(LU + (size_t)ne * ne);
  // row permutation of P A: follow where original row i ends up through the interchanges
  for (int i = tid; i < ne; i += THREADS) {
    int pos = i;
    const int kmax = fail ? fail - 1 : ne;
    for (int k = 0; k < kmax; ++k) {
      const int pr = piv[k];
      if (pos == k) pos = pr;
      else if (pos == pr) pos = k;
    }
    perm[pos] = i;
  }
  if (tid == 0) *info = fail;
  __syncthreads();
}

// Pipeline of the element loop (both roles follow it, meeting at the same barriers):
//   * the next element's A_e and B_e rows of panel q are loaded by TMA as soon as panel q of the current element
//     is finished (those rows of T are dead), one worker warp issuing 16 + 16 row copies at the top of panel
//     q+1; its C_e rows (and the last panel's rows) after the element's last barrier. mbarrier bar[0] counts the
//     first 16 A rows (all the first diagonal block needs), bar[1] everything else.
//   * the chain warp factors the next element's first diagonal block while the workers finish the current
//     element's last panel and store [S | g].
//   * Linv/Uinv buffers alternate on a panel counter that runs across elements.
// GT = true: the working matrix T and the C rows live in this CTA's slab of global scratch (L2-resident) instead of
// shared memory — for elements whose working set exceeds one SM (C5's n_e = 180, 252 buckets). The element's rows
// are then copied in by all threads at its start (no TMA pipeline, no early prologue); everything else is the same
// code on generic pointers.
template <int NWARPS, int MAXT, int MINB, bool GT, bool FUSED>
__global__ void __launch_bounds__(NWARPS * 32, MINB) sweep_kernel(const CondenseArgs a) {
  constexpr int THREADS = NWARPS * 32;
  constexpr int CW = NWARPS - 1;   // the chain warp: the highest warp id wins issue arbitration in its SMSP
  extern __shared__ __align__(128) double smem[];
  const SweepGeo G(a.ne, a.nf);
  const int ne = G.ne, nf = G.nf, ldT = G.ldT, ldC = G.ldC, CB = G.CB, NC = G.NCAB, RA = G.RA;
  const int tid = threadIdx.x, lane = tid & 31;
  // warp index broadcast from lane 0: provably warp-uniform, so the role branches below are not treated as
  // divergent (otherwise every shuffle of the chain warp is wrapped in a collective WARPSYNC loop)
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int gid = lane >> 2, tig = lane & 3;
  const int r1 = ne < NB ? ne : NB;

  double* X = a.scratch + (size_t)blockIdx.x * (size_t)(G.RA * ldT + G.NF8 * ldC);   // exact-path slab
  double* T = GT ? X : smem;
  double* Cr = T + (size_t)RA * ldT;
  double* Linv_b = GT ? smem : Cr + (size_t)G.NF8 * ldC;       // [2][NB * LDI]
  double* Uinv_b = Linv_b + 2 * NB * LDI;          // [2][NB * LDI]
  double* bcast = Uinv_b + 2 * NB * LDI;           // [2][BCW] (spare)
  uint64_t* mbar = reinterpret_cast<uint64_t*>(bcast + 2 * BCW);   // [0] A rows < 16, [1] everything else
  // work-claim counters in the two spare barrier slots: [0..1] trailing blocks, [2..3] TRSM jobs (panel parity)
  int* qctr = reinterpret_cast<int*>(mbar + 2);
  int* piv = reinterpret_cast<int*>(mbar + 4);
  int* sfail = piv + RA;

  for (int i = tid; i < RA * ldT + G.NF8 * ldC; i += THREADS) T[i] = 0.0;
  if (tid == 0) {
    mbar_init(&mbar[0]);
    mbar_init(&mbar[1]);
    for (int i = 0; i < 4; ++i) qctr[i] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  auto elem_of = [&](int64_t it) -> int64_t { return a.elems ? a.elems[it] : it; };
  // one warp: register the next phase's transaction bytes of both barriers
  auto expect_all = [&]() {
    if (lane == 0) {
      mbar_expect_tx(&mbar[0], (uint32_t)(r1 * ne * 8));
      mbar_expect_tx(&mbar[1], (uint32_t)((ne - r1) * ne * 8 + 2 * ne * nf * 8));
    }
    __syncwarp();
  };
  // one warp: A_e and B_e rows [r_lo, r_hi) of element l
  auto load_rows = [&](int64_t l, int r_lo, int r_hi) {
    const double* A = a.A + a.offA[l];
    const double* Bm = a.B + a.offB[l];
    for (int i = r_lo + lane; i < r_hi; i += 32) {
      bulk_g2s(T + (size_t)i * ldT, A + (size_t)i * ne, (uint32_t)(ne * 8), &mbar[i < r1 ? 0 : 1]);
      bulk_g2s(T + (size_t)i * ldT + CB, Bm + (size_t)i * nf, (uint32_t)(nf * 8), &mbar[1]);
    }
  };
  auto load_C = [&](int64_t l) {
    const double* Cm = a.C + a.offC[l];
    for (int i = lane; i < nf; i += 32) bulk_g2s(Cr + (size_t)i * ldC, Cm + (size_t)i * ne, (uint32_t)(ne * 8), &mbar[1]);
  };
  // GT: all threads copy element l's A, B, C rows into the global working slab (16-byte vectors)
  auto stage_global = [&](int64_t l) {
    const double2* A = reinterpret_cast<const double2*>(a.A + a.offA[l]);
    const double2* Bm = reinterpret_cast<const double2*>(a.B + a.offB[l]);
    const double2* Cm = reinterpret_cast<const double2*>(a.C + a.offC[l]);
    const int ha = ne >> 1, hf = nf >> 1;
    const double* sh = a.shift ? a.shift + a.offRe[l] : nullptr;
    for (int q = tid; q < ne * ha; q += THREADS) {
      const int i = q / ha, j = q - i * ha;
      double2 v = __ldg(A + q);
      if (sh && (i >> 1) == j) {   // the diagonal entry of row i is in this pair
        if (i & 1) v.y += __ldg(sh + i);
        else v.x += __ldg(sh + i);
      }
      *reinterpret_cast<double2*>(T + (size_t)i * ldT + 2 * j) = v;
    }
    for (int q = tid; q < ne * hf; q += THREADS) {
      const int i = q / hf, j = q - i * hf;
      *reinterpret_cast<double2*>(T + (size_t)i * ldT + CB + 2 * j) = __ldg(Bm + q);
    }
    for (int q = tid; q < nf * ha; q += THREADS) {
      const int i = q / ha, j = q - i * ha;
      *reinterpret_cast<double2*>(Cr + (size_t)i * ldC + 2 * j) = __ldg(Cm + q);
    }
  };
  // re-condensation: one warp adds element l's diagonal shift to rows [r_lo, r_hi) of T once they have landed
  auto shift_rows = [&](int64_t l, int r_lo, int r_hi) {
    const double* sh = a.shift + a.offRe[l];
    for (int i = r_lo + lane; i < r_hi; i += 32) T[(size_t)i * ldT + i] += __ldg(sh + i);
    __syncwarp();
  };
  auto prefetch = [&](int64_t l) {
    prefetch_l2(a.A + a.offA[l], (uint32_t)(ne * ne * 8));
    prefetch_l2(a.B + a.offB[l], (uint32_t)(ne * nf * 8));
    prefetch_l2(a.C + a.offC[l], (uint32_t)(nf * ne * 8));
    prefetch_l2(a.D + a.offD[l], (uint32_t)(nf * nf * 8));
    // r_e / r_f too: the helper's r_e column and the workers' r_f accumulators are the element's first loads
    // (16-byte granularity: the packed r_e / r_f of an element start 16-byte aligned when n_e, n_f are even)
    if ((a.offRe[l] & 1) == 0) prefetch_l2(a.re + a.offRe[l], (uint32_t)(((ne + 1) & ~1) * 8));
    if ((a.offRf[l] & 1) == 0) prefetch_l2(a.rf + a.offRf[l], (uint32_t)(((nf + 1) & ~1) * 8));
  };

  if (!GT && blockIdx.x < a.count && warp == 0) {
    expect_all();
    load_rows(elem_of(blockIdx.x), 0, ne);
    load_C(elem_of(blockIdx.x));
  }
  uint32_t ph = 0;
  int pc = 0;   // panel counter across elements (Linv/Uinv buffer = pc & 1)

  if (warp == CW) {
    // ======================= chain role: diagonal blocks, their look-ahead TRSM tiles and updates =============
    // One call site of diag_chain / prep_next (code size: the kernel must stay within the instruction cache):
    // panel index -1 is the prologue of an element whose first diagonal block was not factored ahead.
    bool need_pro = true, viol = false;
    for (int64_t it = blockIdx.x; it < a.count; it += gridDim.x, ph ^= 1u) {
      const int64_t l = elem_of(it);
      const int64_t next = it + gridDim.x;
      const int64_t tit = (it - blockIdx.x) / gridDim.x;
      SW_STAMP(tit, 0);
      double* LU = reinterpret_cast<double*>(a.factors + a.offF[l]);
      if constexpr (GT) {
        stage_global(l);
        __syncthreads();   // G: the element is in the global working slab
      }
      bool aborted = false, early = false;
      for (int p = need_pro ? -1 : 0; p < G.npan; ++p) {
        const int jb = p * NB, nb = min(NB, ne - jb), nk = (nb + 3) & ~3;
        const int buf = pc & 1;
        const int jn = jb + NB;
        const bool has_next = jn < ne;
        const int nn = has_next ? min(NB, ne - jn) : 0, nn8 = (nn + 7) & ~7;
        const int nextr_hi = min(jn + NB, RA);
        int jd = 0, nd = r1, dbuf = buf;
        double* LUd = LU;
        bool do_diag = true;
        if (p < 0) {
          if (!GT) {
            mbar_wait(&mbar[0], ph);
            if (a.shift) shift_rows(l, 0, r1);   // the chain warp's first diagonal block: its rows' shift
          }
        } else {
          if (p == 0) SW_STAMP(tit, 110);
          if (__syncthreads_or(viol)) { aborted = true; break; }
          SW_STAMP(tit, 8 + 4 * p);
          viol = false;
          (void)buf;
          named_arrive(1, THREADS);
          SW_STAMP(tit, 9 + 4 * p);
          if (has_next) {
            // the next block's L21 rows / U12 columns come from MMA workers 0 and 1 (their first jobs, off the
            // chain warp's critical path); wait for just those two tiles
            named_sync(2, 96);
            upd_block(T, ldT, T + jb, ldT, T + (size_t)jb * ldT, ldT, jn, nn8 >> 3, jn, nn8 >> 3, nk, lane);
            __syncwarp();
            jd = jn;
            nd = nn;
            dbuf = buf ^ 1;
          } else if (!GT && next < a.count && G.npan >= 2) {
            // the next element's first diagonal block, overlapped with the workers' last-panel work
            // (npan == 1: its rows arrive only after barrier F)
            mbar_wait(&mbar[0], ph ^ 1u);
            if (a.shift) shift_rows(elem_of(next), 0, r1);
            LUd = reinterpret_cast<double*>(a.factors + a.offF[elem_of(next)]);
            dbuf = buf ^ 1;
            early = true;
          } else {
            do_diag = false;
          }
          SW_STAMP(tit, 10 + 4 * p);
        }
        if (do_diag)
          viol |= diag_block<GT>(T, ldT, jd, nd, Linv_b + dbuf * NB * LDI, Uinv_b + dbuf * NB * LDI, bcast, LUd, ne, lane);
        if (p < 0) {
          SW_STAMP(tit, 2);
          if (!GT) mbar_wait(&mbar[1], ph);
          SW_STAMP(tit, 3);
        } else {
          SW_STAMP(tit, 11 + 4 * p);
          ++pc;
        }
      }
      SW_STAMP(tit, 100);
      need_pro = !early;
      if (aborted) {
        ++pc;   // the aborted panel's buffer may be half-written
        __syncthreads();   // A: remaining loads of the next element issued by the loader warp
        {
          const SgDst d = sg_dst(a, l);
          exact_element<THREADS>(d.S, d.g, d.Kf, d.Ef, d.eblk, d.eE, d.so, a.A + a.offA[l], a.B + a.offB[l],
                                 a.re + a.offRe[l], a.C + a.offC[l], a.D + a.offD[l], a.rf + a.offRf[l],
                                 a.shift ? a.shift + a.offRe[l] : nullptr,
                                 reinterpret_cast<double*>(a.factors + a.offF[l]), a.info + l, ne, nf, X, piv, sfail,
                                 tid);
        }
      } else {
        SW_STAMP(tit, 6);
        __syncthreads();   // E: every read of T / Cr of this element is done
        SW_STAMP(tit, 7);
      }
      SW_STAMP(tit, 101);
    }
  } else {
    // ======================= worker role: TRSM tiles, trailing updates, register-resident [S | g] ============
    // DMMA throughput is per SMSP (one m8n8k4 per 16 cycles per warp scheduler), so the warp sharing the chain
    // warp's SMSP (warp HW = CW - 4) issues no MMAs — it is the helper (r_e column, TMA loads of the next
    // element, permutation/info); the NWK = NWARPS - 2 MMA workers live on the other SMSPs.
    constexpr int HW = CW - 4;
    constexpr int NWK = NWARPS - 2;
    const bool helper = warp == HW;
    const int w = warp < HW ? warp : warp - 1;   // MMA worker index 0 .. NWK-1 (unused for the helper)
    // GT: dynamic work claiming, one shared-memory atomic per job broadcast to the warp (the jobs' run times vary
    // with L2 hits: C5 slab 90.3 -> 88.4 ms). Shared-memory T: static round-robin (dynamic measured 38.6 -> 39.0 ms
    // on C4: equal-cost jobs, the atomic is pure latency)
    auto claim = [&](int* c) -> int {
      int v = 0;
      if (lane == 0) v = atomicAdd(c, 1);
      return __shfl_sync(0xffffffffu, v, 0);
    };
    double acc[MAXT][2];
    // fixed shared-memory offsets of this worker's [S | g] tiles: Y rows (Cr) and W columns (T); slots past the
    // last tile accumulate into dead registers
    // offD[s]: D_e offset of this lane's accumulator pair (>= 0), -(row + 2) for the r_f column, -1 for padding
    int offY[MAXT], offW[MAXT], offD[MAXT];
    // row map: when the [S | g] tile rows are exactly the MMA workers and a row's column tiles fill the slots (C4:
    // 6 x 7 tiles), worker w owns tile row w, so one Y_p fragment per k-step serves all its slots (8 shared loads
    // per 7 DMMAs instead of 14); otherwise tiles are dealt round-robin
    const bool rowmap = G.NF8 / 8 == NWK && G.CTs == MAXT && !(a.debug & 8);
#pragma unroll
    for (int s = 0; s < MAXT; ++s) {
      const int t0 = rowmap ? w * MAXT + s : w + s * NWK;
      const int t = min(t0, G.ntiles - 1);
      const int row = (t / G.CTs) * 8 + gid, c = (t % G.CTs) * 8 + 2 * tig;
      offY[s] = row * ldC + tig;
      offW[s] = CB + (t % G.CTs) * 8 + gid + tig * ldT;
      offD[s] = (t0 < G.ntiles && row < nf) ? (c < nf ? row * nf + c : (c == nf ? -(row + 2) : -1)) : -1;
    }
    double rv[(kMaxNe + 31) / 32];   // helper: the next element's r_e column, loaded ahead
    bool have_rv = false, have_acc = false;
    // the accumulators from D_e / r_f (precomputed offsets: no divisions, no branches around the loads)
    auto load_acc = [&](int64_t le) {
      const double* D = a.D + a.offD[le];
      const double* rf = a.rf + a.offRf[le];
#pragma unroll
      for (int s = 0; s < MAXT; ++s) {
        const int o = offD[s];
        const double2 v = __ldg(reinterpret_cast<const double2*>(D + (o >= 0 ? o : 0)));
        const double r0v = __ldg(rf + (o < -1 ? -o - 2 : 0));
        acc[s][0] = o >= 0 ? v.x : (o < -1 ? r0v : 0.0);
        acc[s][1] = o >= 0 ? v.y : 0.0;
      }
    };
    for (int64_t it = blockIdx.x; it < a.count; it += gridDim.x, ph ^= 1u) {
      const int64_t l = elem_of(it);
      const int64_t next = it + gridDim.x;
      const int64_t ln = next < a.count ? elem_of(next) : -1;
      const int64_t tit = (it - blockIdx.x) / gridDim.x;
      SW_STAMP(tit, 0);
      double* LU = reinterpret_cast<double*>(a.factors + a.offF[l]);
      if constexpr (GT) {
        stage_global(l);
        __syncthreads();   // G
      }
      if (helper) {
        // (the next element's L2 prefetch is issued at panel 1, behind the TMA row copies: issued here, right after
        // the previous element's last row / C-row copies, it held the helper ~8 K cycles at the first barrier)
        if (GT && lane == 0 && ln >= 0) prefetch(ln);
        // the r_e column: every load issued before the first shared store (the generic T pointer could alias the
        // global input as far as the compiler knows: interleaved load/store pairs serialise on the HBM latency —
        // measured, the helper reached the first panel barrier 3-6 K cycles after the workers)
        // (loaded before the previous element's last barrier when there was one: its HBM latency then overlaps the
        // end of that element instead of holding the first panel barrier)
        if (!have_rv) {
          const double* re = a.re + a.offRe[l];
#pragma unroll
          for (int q = 0; q < (kMaxNe + 31) / 32; ++q) rv[q] = lane + 32 * q < ne ? __ldg(re + lane + 32 * q) : 0.0;
        }
        have_rv = false;
#pragma unroll
        for (int q = 0; q < (kMaxNe + 31) / 32; ++q)
          if (lane + 32 * q < ne) T[(size_t)(lane + 32 * q) * ldT + CB + nf] = rv[q];
      } else {
        if (!have_acc) load_acc(l);
        have_acc = false;
      }
      SW_STAMP(tit, 4);
      if (!GT) mbar_wait(&mbar[0], ph);
      SW_STAMP(tit, 5);
      if (!GT) mbar_wait(&mbar[1], ph);
      if (!GT && a.shift && helper) shift_rows(l, r1, ne);   // before the first panel barrier: no reader yet
      SW_STAMP(tit, 3);
      bool viol = false;
      bool aborted = false;
      int p_ab = G.npan;
      for (int p = 0; p < G.npan; ++p, ++pc) {
        if (p == 0) SW_STAMP(tit, 110);
        if (helper && p == 0 && a.trace && blockIdx.x == 0 && tit < 4 && lane == 0) a.trace[tit * 256 + 112] = clock64();
        if (__syncthreads_or(viol)) { aborted = true; p_ab = p; break; }
        SW_STAMP(tit, 8 + 4 * p);
        viol = false;
        // the next panel's counters: their last users (the previous panel) have all passed the barrier above
        if (GT && helper && lane == 0) qctr[(pc + 1) & 1] = qctr[2 + ((pc + 1) & 1)] = 0;
        if (GT && helper && p >= 1 && !(a.debug & 16)) {
          // the slab rows of panel p-1 are dead for the rest of the element (their L\U is in the factor record,
          // their U12 / W parts were last read by panel p-1's updates): drop their L2 lines without a write-back
          // (only lines entirely inside those rows; the next element's staging rewrites them)
          const uintptr_t lo = ((uintptr_t)(T + (size_t)(p - 1) * NB * ldT) + 127) & ~(uintptr_t)127;
          const uintptr_t hi = (uintptr_t)(T + (size_t)min(p * NB, ne) * ldT) & ~(uintptr_t)127;
          for (uintptr_t q = lo + 128 * (uintptr_t)lane; q < hi; q += 128 * 32) discard_l2_line((const void*)q);
        }
        if (!GT && helper && p >= 1 && ln >= 0) {
          // the rows of panel p-1 are dead: stream the next element's rows in
          if (p == 1) expect_all();
          fence_proxy_async();
          load_rows(ln, (p - 1) * NB, p * NB);
          if (p == 1 && lane == 0) prefetch(ln);
        }
        // one panel step; NBC = 16: a full panel, every size below is a compile-time constant (no guards around
        // the fragment loads, so they are scheduled ahead of the DMMAs); NBC = 0: the partial last panel
        auto body = [&](auto nbc) {
          constexpr int NBC = decltype(nbc)::value;
          const int jb = p * NB;
          const int nb = NBC ? NBC : min(NB, ne - jb);
          const int nk = (nb + 3) & ~3, nb8 = (nb + 7) & ~7;
          const int buf = pc & 1;
          const double* Linv = Linv_b + buf * NB * LDI;
          const double* Uinv = Uinv_b + buf * NB * LDI;
          const int jn = jb + NB;
          const bool has_next = jn < ne;
          const int nn = has_next ? min(NB, ne - jn) : 0, nn8 = (nn + 7) & ~7;
          const int nextr_hi = min(jn + NB, RA);
          // ---- TRSM tiles: L21 (A rows below the next panel), Y_p (C rows), U12 (columns), two tiles per job
          const int rA0 = has_next ? nextr_hi : RA;                 // A rows [rA0, RA)
          const int cU0 = has_next ? jn + nn8 : jb + nb8;           // columns [cU0, NC)
          const int tA = (RA - rA0) >> 3, tC = G.NF8 >> 3, tU = (NC - cU0) >> 3;
          const int nA = (tA + 1) >> 1, nCt = (tC + 1) >> 1, nU = (tU + 1) >> 1;
          if (has_next && w < 2 && !helper) {
            // the tiles the chain warp's next diagonal block needs, first: L21 of its rows, U12 of its columns
            if (w == 0) viol |= trsm_right<GT>(T, ldT, jn, (nextr_hi - jn) >> 3, jb, nb, Uinv, ne, LU, lane);
            else trsm_left<GT>(T, ldT, jb, nb, Linv, jn, nn8 >> 3, LU, ne, lane);
            __syncwarp();
            named_arrive(2, 96);
          }
          // regular jobs start from worker 2: workers 0 and 1 (which also carry the look-ahead tiles) get the
          // remainder jobs last
          // (measured: the helper taking regular jobs too in the first two thirds of the panels — 7 takers — made
          //  C4 2.2 ms slower: its DMMAs on the chain warp's SMSP land during the chain's diagonal block; re-measured
          //  with the helper's own trailing share, its last 1-3 jobs in the first 2-6 panels only: 34.3-36.0 vs 34.05 ms)
          for (int job = ((a.debug & 1) || helper) ? 1 << 30 : (GT ? claim(qctr + 2 + (pc & 1)) : (w + NWK - 2) % NWK);
               job < nA + nCt + nU; job = GT ? claim(qctr + 2 + (pc & 1)) : job + NWK) {
            if (job < nA) {
              viol |= trsm_right<GT>(T, ldT, rA0 + 16 * job, min(2, tA - 2 * job), jb, nb, Uinv, ne, LU, lane);
            } else if (job < nA + nCt) {
              const int q = job - nA;
              trsm_right<GT>(Cr, ldC, 16 * q, min(2, tC - 2 * q), jb, nb, Uinv, 0, nullptr, lane);
            } else {
              const int q = job - nA - nCt;
              trsm_left<GT>(T, ldT, jb, nb, Linv, cU0 + 16 * q, min(2, tU - 2 * q), LU, ne, lane);
            }
          }
          named_sync(1, THREADS);
          SW_STAMP(tit, 9 + 4 * p);
          // ---- register-resident [S | g] -= Y_p W_p
          if (!helper) {
            const double* Yp = Cr + jb;
            const double* Wp = T + (size_t)jb * ldT;
            if (rowmap) {
#pragma unroll
              for (int k = 0; k < NB; k += 4) {
                if (k < nk && !(a.debug & 2)) {
                  const double y = -Yp[offY[0] + k];
#pragma unroll
                  for (int s = 0; s < MAXT; ++s) dmma(acc[s], y, Wp[offW[s] + k * ldT]);
                }
              }
            } else {
#pragma unroll
              for (int k = 0; k < NB; k += 4) {
                if (k < nk && !(a.debug & 2)) {
#pragma unroll
                  for (int s = 0; s < MAXT; ++s) dmma(acc[s], -Yp[offY[s] + k], Wp[offW[s] + k * ldT]);
                }
              }
            }
          }
          SW_STAMP(tit, 10 + 4 * p);
          // ---- trailing updates: R1a (rows of the next panel, right of its diagonal block), R1b (A rows
          //      below), R2 (C rows over A columns)
          if (has_next) {
            const Region R1a(jn, nextr_hi, jn + nn8, NC);
            const Region R1b(nextr_hi, RA, jn, NC);
            const Region R2(0, G.NF8, jn, CB);
            const int tot = R1a.nblk + R1b.nblk + R2.nblk;
            // trailing blocks: the 6 MMA workers, plus the helper in the first two thirds of the panels (there the
            // workers bound the step; later the chain warp does, and it shares the helper's SMSP tensor pipe)
            const bool hjoin = 3 * p < 2 * G.npan;   // (first 2/3: C4 38.7 -> 38.4 ms vs the first half)
            const int nt_w = hjoin ? NWK + 1 : NWK;
            const int tw = helper ? NWK : w;
            // Shared-memory T: the helper takes the LAST kHelperShare/64 of the blocks one after another (mostly the
            // C-row blocks of R2, starting while the workers still update [S | g]) and the workers deal the rest
            // round-robin. Measured on C4 in
            // one binary (HDG_DEBUG_MODE bits 8-13 override the share; 1 = the previous 7-taker interleaved deal):
            // interleaved 35.1-35.3 ms, share 10: 35.0, 12: 34.4, 13: 34.3, 14: 34.0-34.4, 15: 34.4, 16: 35.7,
            // 18: 37.6 ms; joining in more or fewer panels, or rounding the workers' share to whole rounds: no gain.
            // (Also measured, not adopted: the C rows on an mbarrier of their own, waited for at their first use in
            // panel 0 with the Y_p jobs dealt last — 34.5-34.7 vs 34.05 ms: the element start is not bound by them.)
            const int hsel = ((a.debug >> 8) & 63) ? (a.debug >> 8) & 63 : kHelperShare;
            const int nh = (!GT && hjoin && hsel > 1) ? (tot * hsel) >> 6 : -1;
            const int b_end = (nh >= 0 && !helper) ? tot - nh : tot;
            const int b0 = nh >= 0 ? (helper ? tot - nh : w) : tw;
            const int bs = nh >= 0 ? (helper ? 1 : NWK) : nt_w;
            for (int b = ((a.debug & 1) || (helper && !hjoin)) ? 1 << 30 : (GT ? claim(qctr + (pc & 1)) : b0); b < b_end;
                 b = GT ? claim(qctr + (pc & 1)) : b + bs) {
              // region selection with plain integers (no addresses of locals: they would live on the stack)
              int bi = b, r_lo, r_hi, c_lo, c_hi, nbc;
              const bool inC = bi >= R1a.nblk + R1b.nblk;
              if (bi < R1a.nblk) { r_lo = R1a.r_lo; r_hi = R1a.r_hi; c_lo = R1a.c_lo; c_hi = R1a.c_hi; nbc = R1a.nbc; }
              else if ((bi -= R1a.nblk) < R1b.nblk) { r_lo = R1b.r_lo; r_hi = R1b.r_hi; c_lo = R1b.c_lo; c_hi = R1b.c_hi; nbc = R1b.nbc; }
              else { bi -= R1b.nblk; r_lo = R2.r_lo; r_hi = R2.r_hi; c_lo = R2.c_lo; c_hi = R2.c_hi; nbc = R2.nbc; }
              double* dst = inC ? Cr : T;
              const int ldd = inC ? ldC : ldT;
              // block row by a fast float division ((bi + 0.5) / nbc is >= 1/16 from an integer for bi < 1024,
              // nbc <= 8, far beyond __fdividef's error): ncu put 5 % of the stall samples on the integer division
              // in front of every block's fragment loads (A/B in one binary: C4 condense 36.19 -> 35.39 ms)
              const int br = (int)__fdividef((float)bi + 0.5f, (float)nbc), bc = bi - br * nbc;
              const int r0 = r_lo + 16 * br, c0 = c_lo + 32 * bc;
              const int nrt = min(2, (r_hi - r0) >> 3), nct = min(4, (c_hi - c0) >> 3);
              if (nrt == 2 && nct == 4 && NBC == NB) upd_full16(dst, ldd, dst + jb, ldd, T + (size_t)jb * ldT, ldT, r0, c0, lane);
              else if (nrt == 2 && nct == 4) upd_block(dst, ldd, dst + jb, ldd, T + (size_t)jb * ldT, ldT, r0, 2, c0, 4, nk, lane);
              else upd_block(dst, ldd, dst + jb, ldd, T + (size_t)jb * ldT, ldT, r0, nrt, c0, nct, nk, lane);
            }
          }
          SW_STAMP(tit, 11 + 4 * p);
        };
        if ((p + 1) * NB <= ne) body(std::integral_constant<int, NB>{});
        else body(std::integral_constant<int, 0>{});
      }
      SW_STAMP(tit, 100);
      if (aborted) {
        ++pc;
        // issue every load of the next element that is not in flight yet (its rows of T are dead), then redo
        // this element on the exact path in global scratch
        if (!GT && ln >= 0 && helper) {
          if (p_ab <= 1) expect_all();
          fence_proxy_async();
          load_rows(ln, p_ab >= 1 ? (p_ab - 1) * NB : 0, ne);
          load_C(ln);
        }
        __syncthreads();   // A
        if (helper && lane == 0) qctr[0] = qctr[1] = qctr[2] = qctr[3] = 0;   // (the exact path's barriers order it)
        {
          const SgDst d = sg_dst(a, l);
          exact_element<THREADS>(d.S, d.g, d.Kf, d.Ef, d.eblk, d.eE, d.so, a.A + a.offA[l], a.B + a.offB[l],
                                 a.re + a.offRe[l], a.C + a.offC[l], a.D + a.offD[l], a.rf + a.offRf[l],
                                 a.shift ? a.shift + a.offRe[l] : nullptr,
                                 reinterpret_cast<double*>(a.factors + a.offF[l]), a.info + l, ne, nf, X, piv, sfail,
                                 tid);
        }
      } else {
        // every worker is past its last read of T / Cr once the last panel's [S | g] update is done: the helper
        // issues the next element's remaining rows and C rows then, ahead of the [S | g] stores and barrier E
        // (debug bit 26: after E as before; bit 27: the next D_e / r_f accumulators loaded at the element start).
        // Measured on C4 in one binary: both 33.6 ms, early loads alone 34.65, early accumulators alone 35.4,
        // neither 34.05 ms — the element start waits for whichever of the two lands last.
        const bool eload = !GT && ln >= 0 && !(a.debug & (1 << 26));
        if (eload) {
          if (helper) {
            named_sync(3, (NWK + 1) * 32);
            if (G.npan == 1) expect_all();
            fence_proxy_async();
            load_rows(ln, (G.npan - 1) * NB, ne);
            load_C(ln);
          } else {
            named_arrive(3, (NWK + 1) * 32);
          }
        }
        if (helper) {
          int32_t* perm = reinterpret_cast<int32_t*>(LU + (size_t)ne * ne);
          for (int i = lane; i < ne; i += 32) perm[i] = i;
          if (lane == 0) a.info[l] = 0;
          if (!GT && ln >= 0) {   // the next element's r_e column, landing while the workers store [S | g]
            const double* re = a.re + a.offRe[ln];
#pragma unroll
            for (int q = 0; q < (kMaxNe + 31) / 32; ++q) rv[q] = lane + 32 * q < ne ? __ldg(re + lane + 32 * q) : 0.0;
            have_rv = true;
          }
        } else {
          if constexpr (FUSED) {   // hdg_condense_assemble: straight into K, E
            const SgDst dst = sg_dst(a, l);
#pragma unroll
            for (int s = 0; s < MAXT; ++s) {
              const int o = offD[s];
              if (o >= 0) out_S2(dst, nf, o / nf, o - (o / nf) * nf, acc[s][0], acc[s][1]);
              else if (o < -1) out_g(dst, -o - 2, acc[s][0]);
            }
          } else {
            double* S = a.S + a.offS[l];
            double* g = a.g + a.offG[l];
#pragma unroll
            for (int s = 0; s < MAXT; ++s) {
              const int o = offD[s];
              if (o >= 0) st_lu<GT>(S + o, acc[s][0], acc[s][1]);
              else if (o < -1) g[-o - 2] = acc[s][0];
            }
          }
          if (!GT && ln >= 0 && !(a.debug & (1 << 27))) {   // the next element's accumulators, landing across E
            load_acc(ln);
            have_acc = true;
          }
        }
        SW_STAMP(tit, 6);
        __syncthreads();   // E: every read of T / Cr of this element is done
        SW_STAMP(tit, 7);
        if (!GT && ln >= 0 && helper && !eload) {
          if (G.npan == 1) expect_all();
          fence_proxy_async();
          load_rows(ln, (G.npan - 1) * NB, ne);
          load_C(ln);
        }
        // no barrier here: the workers wait for these rows on the mbarrier's transaction count, the chain warp at
        // the next element's first panel barrier (a CTA barrier here measured 0.4 ms slower on C4)
      }
      SW_STAMP(tit, 101);
    }
  }
}

template <int NWARPS, int MAXT, int MINB, bool GT>
cudaError_t launch_sweep_t(const CondenseArgs& a, int sms, cudaStream_t s) {
  const SweepGeo G(a.ne, a.nf);
  const int64_t smem = GT ? G.smem_bytes() - 8 * ((int64_t)G.RA * G.ldT + (int64_t)G.NF8 * G.ldC) : G.smem_bytes();
  auto kern = a.Kf ? sweep_kernel<NWARPS, MAXT, MINB, GT, true> : sweep_kernel<NWARPS, MAXT, MINB, GT, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NWARPS * 32, (size_t)smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = (int64_t)sms * (per_sm < 2 ? per_sm : 2);   // the exact-path scratch holds 2 slabs per SM
  if (GT) {
    // one CTA per SM. Capping the slabs to keep them all L2-resident was measured slower on C5 (80 MB of slabs:
    // 114 ms, all 148 SMs with 121 MB of slabs: 106 ms); HDG_GT_L2_MB still sets a cap for experiments
    const int64_t slab = 8 * ((int64_t)G.RA * G.ldT + (int64_t)G.NF8 * G.ldC);
    const char* lb = getenv("HDG_GT_L2_MB");
    grid = lb ? std::min<int64_t>(sms, std::max<int64_t>(1, atoll(lb) * 1024 * 1024 / slab)) : sms;
  }
  if (grid > a.count) grid = a.count;
  grid = grid_cap(grid);
  kern<<<(unsigned)grid, NWARPS * 32, (size_t)smem, s>>>(a);
  return cudaGetLastError();
}

// The exact path over a device-side list of elements (the row-tile kernel's failed speculations): one element
// per CTA at a time in the CTA's global scratch slab; the list length is read on the device (0: immediate exit).
template <int THREADS>
__global__ void __launch_bounds__(THREADS) exact_list_kernel(const CondenseArgs a, const int32_t* list,
                                                             const int32_t* count) {
  extern __shared__ __align__(16) int ish[];
  const SweepGeo G(a.ne, a.nf);
  int* piv = ish;
  int* sfail = ish + G.RA;
  double* X = a.scratch + (size_t)blockIdx.x * (size_t)(G.RA * G.ldT + G.NF8 * G.ldC);
  const int n = *count;
  for (int q = blockIdx.x; q < n; q += gridDim.x) {
    const int64_t l = list[q];
    const SgDst d = sg_dst(a, l);
    exact_element<THREADS>(d.S, d.g, d.Kf, d.Ef, d.eblk, d.eE, d.so, a.A + a.offA[l], a.B + a.offB[l],
                           a.re + a.offRe[l], a.C + a.offC[l], a.D + a.offD[l], a.rf + a.offRf[l],
                           a.shift ? a.shift + a.offRe[l] : nullptr,
                           reinterpret_cast<double*>(a.factors + a.offF[l]), a.info + l, a.ne, a.nf, X, piv, sfail,
                           threadIdx.x);
  }
}

}  // namespace

cudaError_t launch_exact_list(const CondenseArgs& a, const int32_t* list, const int32_t* count, int grid, cudaStream_t s) {
  const SweepGeo G(a.ne, a.nf);
  const size_t smem = sizeof(int) * (G.RA + 4);
  exact_list_kernel<256><<<(unsigned)std::max(1, grid), 256, smem, s>>>(a, list, count);
  return cudaGetLastError();
}

// Whether the sweep kernel with T in shared memory handles (ne, nf).
bool sweep_supported(int ne, int nf, size_t smem_optin) {
  const SweepGeo G(ne, nf);
  if ((size_t)G.smem_bytes() > smem_optin) return false;
  return (G.ntiles + 5) / 6 <= 16;
}
// Whether the global-slab variant handles it (elements larger than one SM: n_e <= 256, [S | g] in <= 16 slots).
bool sweep_gt_supported(int ne, int nf) {
  const SweepGeo G(ne, nf);
  return ne <= kMaxNe && (G.ntiles + 5) / 6 <= 16;
}

cudaError_t launch_condense_sweep_gt(const CondenseArgs& a, int sms, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  ++*launches;
  const SweepGeo G(a.ne, a.nf);
  // 16 warps (14 MMA workers, 4 per SMSP): the L2 latency of the slab's fragment loads needs the extra warps
  // (C5 slab measured 107 -> 92 ms vs 8 warps; 12 warps: 99 ms). The shared-memory sweep keeps 8 (C4: 42.9 vs
  // 47.2 ms with 16 — its chain warp, not load latency, bounds it). Caching T's bottom rows in the free shared
  // memory was measured slower (the 252 bucket 36 -> 41 ms): it takes the L1 capacity that already holds the
  // slab's re-read fragments.
  if ((G.ntiles + 13) / 14 <= 7) return launch_sweep_t<16, 7, 1, true>(a, sms, s);
  const int slots = (G.ntiles + 5) / 6;
  if (slots <= 11) return launch_sweep_t<8, 11, 1, true>(a, sms, s);
  return launch_sweep_t<8, 16, 1, true>(a, sms, s);
}

cudaError_t launch_condense_sweep(const CondenseArgs& a, int sms, size_t smem_optin, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  ++*launches;
  const SweepGeo G(a.ne, a.nf);
  (void)smem_optin;
  const int slots = (G.ntiles + 5) / 6;
  // two CTAs (two elements, two chain warps) per SM when their shared memory fits: the 128-register build has no
  // spills up to 12 [S|g] slots (checked with -Xptxas -v), and the second element hides the first's chain latency
  const bool two = 2 * (G.smem_bytes() + 1024) <= 233472 && slots <= 12;
  if (two) {
    if (slots <= 4) return launch_sweep_t<8, 4, 2, false>(a, sms, s);
    if (slots <= 7) return launch_sweep_t<8, 7, 2, false>(a, sms, s);
    return launch_sweep_t<8, 12, 2, false>(a, sms, s);
  }
  if (slots <= 4) return launch_sweep_t<8, 4, 1, false>(a, sms, s);
  if (slots <= 7) return launch_sweep_t<8, 7, 1, false>(a, sms, s);
  if (slots <= 11) return launch_sweep_t<8, 11, 1, false>(a, sms, s);
  return launch_sweep_t<8, 16, 1, false>(a, sms, s);
}

}  // namespace hdg
