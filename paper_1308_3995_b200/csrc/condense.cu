// condense.cu — rows a1-a5 of the hot path: element-local static condensation.
//
// For each element e (Eq. hybridsystem; "condense"):
//     S_e = D_e - C_e A_e^-1 B_e,   g_e = r_f - C_e A_e^-1 r_e,
// with A_e factored by Gaussian elimination with partial pivoting (GEPP) and the factorization
// kept for the reconstruction.
//
// One CTA owns one element at a time (persistent grid). The working matrix T = [A_e | 0 | B_e | r_e | 0]
// (rows padded with zeros to a multiple of 16) lives in shared memory, or in an L2-resident global scratch slab
// when it does not fit (hp degrees p >= 4).
//
//   phase A  : blocked right-looking elimination of the A rows across all columns, panels of kNB = 16:
//              T <- [L\U | L^-1 P B | L^-1 P r_e].
//              Fast path (speculative GEPP): the 16x16 diagonal block is factored by one warp in natural order
//              and inverted (L11^-1, U11^-1); L21 = A21 U11^-1, U12 = L11^-1 A12 and the trailing update
//              A22 -= L21 U12 all run on the FP64 tensor cores (DMMA m8n8k4). Every multiplier is checked:
//              if any |l_ik| > 1 (or a pivot is 0), partial pivoting would have interchanged rows, and the
//              element is re-staged and redone on the pivoting path. When the check passes, the pivot sequence
//              of GEPP is the identity and this IS GEPP.
//              Pivoting path: one warp factors the whole panel column by column with the GEPP pivot search
//              (maximal |a_ik|, lowest index on ties), interchanges are applied to the
//              other columns, then U12 and the trailing update as above.
//   factors  : L\U written row-major + the row permutation (for hdg_backsubstitute).
//   phase A' : X = U^-1 [L^-1 P B | L^-1 P r_e] = A_e^-1 [B_e | r_e] by blocked backward substitution, panels
//              bottom-up: X_p = U_pp^-1 W_p and W_<p -= U_<p,p X_p, both DMMA.
//   phase B  : [S_e | g_e] = [D_e | r_f] - C_e X, DMMA GEMM n_f x (n_f+1) x n_e per element; C_e, D_e read from
//              HBM straight into fragments, S_e, g_e stored straight to HBM.
// FLOPs: SURVEY.md §8(d)'s algorithmic count n_e(n_e-1)(4n_e+1)/6 + (n_f+1)(2n_e^2-n_e) + 2 n_f n_e (n_f+1)
// plus the O(16 n_e^2) explicit 16x16 inverse applications.
#include "hdg_internal.cuh"

namespace hdg {
namespace {

constexpr int NB = kNB;   // 16

// instrumentation: stamp k of element-iteration `it` (CTA 0, first 4 elements), per warp 0 / warp 1
#define HDG_STAMP(trace, it, k)                                                                          \
  do {                                                                                                   \
    if ((trace) && blockIdx.x == 0 && (it) < 4 && (threadIdx.x == 0 || threadIdx.x == 32))               \
      (trace)[(it) * 256 + (threadIdx.x >> 5) * 128 + (k)] = clock64();                                  \
  } while (0)
constexpr int LDI = 20;   // row stride of the 16x16 inverse buffers (= 4 mod 16: conflict-free fragments)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// Row order of accumulator tiles and their A operands: accumulator row g <-> T row srow(g) (bits 0 and 1 of g
// swapped), so the 16-byte accumulator accesses of a quarter warp (two rows) fall in opposite halves of the bank
// space with the row stride Geo picks (4 mod 16 doubles, which keeps the 8-byte fragment loads conflict-free);
// A rows and accumulator rows are permuted together, the product is unchanged (same fix as condense_sweep.cu).
__device__ __forceinline__ int srow(int g) { return (g & 4) | ((g & 1) << 1) | ((g >> 1) & 1); }

// dst[r][c] -= sum_{k < nk} As[r][k] * Bs[k][c] over rows [r_lo, r_hi) (multiples of 16) and columns
// [c_lo, c_hi) (multiples of 8); nk multiple of 4. dst, As, Bs share the row stride ld. Work unit: a 16 x 32
// block (2 x 4 tiles of 8x8) per warp, so each k-step loads 2 A- and 4 B-fragments for 8 DMMAs and every
// accumulator tile is read and written once per call. Blocks are numbered row-major; this warp takes blocks
// first, first + stride, ... (at most max_blocks of them).
__device__ __forceinline__ void mma_update(double* dst, const double* As, const double* Bs, int ld, int r_lo, int r_hi,
                                           int c_lo, int c_hi, int nk, int first, int stride, int lane,
                                           int max_blocks = 1 << 30) {
  const int BR = (r_hi - r_lo) >> 4, CT = (c_hi - c_lo) >> 3;
  if (BR <= 0 || CT <= 0) return;
  const int BC = (CT + 3) >> 2;
  const int nblk = min(BR * BC, max_blocks);
  const int gid = lane >> 2, tig = lane & 3, sg = srow(gid);
  for (int blk = first; blk < nblk; blk += stride) {
    const int br = blk / BC, bc = blk - br * BC;
    const int r0 = r_lo + br * 16, c0 = c_lo + bc * 32;
    const int nct = min(4, CT - 4 * bc);
    double acc[2][4][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[i][j][0] = 0.0;
        acc[i][j][1] = 0.0;
        if (j < nct) {
          const double2 v = *reinterpret_cast<const double2*>(dst + (r0 + 8 * i + sg) * ld + c0 + 8 * j + 2 * tig);
          acc[i][j][0] = v.x;
          acc[i][j][1] = v.y;
        }
      }
    for (int k = 0; k < nk; k += 4) {
      const double a0 = -As[(r0 + sg) * ld + k + tig];
      const double a1 = -As[(r0 + 8 + sg) * ld + k + tig];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j < nct) {
          const double b = Bs[(k + tig) * ld + c0 + 8 * j + gid];
          dmma(acc[0][j], a0, b);
          dmma(acc[1][j], a1, b);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < nct)
          *reinterpret_cast<double2*>(dst + (r0 + 8 * i + sg) * ld + c0 + 8 * j + 2 * tig) =
              make_double2(acc[i][j][0], acc[i][j][1]);
  }
}

// Phase A' for one column tile (8 columns at c0) of W, entirely inside one warp (no CTA barriers): panels
// bottom-up, X_p = U_pp^-1 W_p, then W_<p -= U_<p,p X_p for this tile only.
__device__ __forceinline__ void backsolve_tile(double* T, int ldT, int ne, const double* Uinv_all, int c0, int lane);

// 1/x with one MUFU.RCP64H and two Newton steps (no slow path; pivots here are finite and non-zero, a zero or
// non-finite pivot is caught by the GEPP speculation check and redone on the pivoting path).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;\n" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Fast path: factor the 16x16 diagonal block at (jb, jb) in natural row order and invert both factors, one
// warp. A partial block (nb < 16, last panel) is padded with identity rows/columns, so L11^-1 and U11^-1 carry
// ones on the padded diagonal (harmless: the padded rows/columns of T are zero).
//   forward:  lane r < 16 holds row r in registers; step c broadcasts the pivot row (shuffles), every lower row
//             forms its multiplier and updates itself -> L\U (written back to T, rows < nb only);
//   inverses: lane c < 16 solves L x = e_c (column c of L11^-1); lane 16 + c solves the index-reversed lower
//             system J U J z = e_(15-c) (column c of U11^-1 = J z); one instruction stream, lane-dependent
//             addresses, right-looking substitution with the factors read from T (broadcast loads).
// Linv/Uinv: row-major 16x16, stride LDI. Returns true if GEPP would have interchanged rows (|a_ik| > |a_kk|,
// i > k) or a pivot is zero.
__device__ __forceinline__ bool diag_factor(double* T, int ldT, int jb, int nb, double* Linv, double* Uinv, int lane) {
  double d[NB];
  double* rcs = Linv + NB * LDI;   // 16 pivot reciprocals (shared memory: keeps them out of the register file)
  const bool real = lane < nb;
  double* Dg = T + jb * ldT + jb;
  const double2* src = reinterpret_cast<const double2*>(Dg + (real ? lane : 0) * ldT);
#pragma unroll
  for (int j = 0; j < NB; j += 2) {
    double2 v = make_double2(j == lane ? 1.0 : 0.0, j + 1 == lane ? 1.0 : 0.0);   // identity padding
    if (real) v = src[j / 2];
    d[j] = v.x;
    d[j + 1] = v.y;
  }
  bool viol = false;
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    double prow[NB];
#pragma unroll
    for (int j = c; j < NB; ++j) prow[j] = __shfl_sync(0xffffffffu, d[j], c);
    const double pv = prow[c];
    viol |= !(fabs(pv) >= 2.2250738585072014e-308) || !(fabs(pv) < 1.0e300);   // zero/subnormal/huge/NaN: exact path (R7, R16)
    const double rp = fast_rcp(pv);
    if (lane == 0) rcs[c] = rp;
    if (lane > c && lane < NB) {
      viol |= fabs(d[c]) > fabs(pv);
      const double l = d[c] * rp;
      d[c] = l;
#pragma unroll
      for (int j = c + 1; j < NB; ++j) d[j] = fma(-l, prow[j], d[j]);
    }
  }
  // the identity-padded factors go to a scratch copy of the block (Linv's storage is reused after), T gets
  // only the real rows
  double* F = Uinv;   // 16 x LDI scratch: overwritten by U^-1 below, after all lanes have read it
  if (lane < NB) {
    double2* dst = reinterpret_cast<double2*>(F + lane * LDI);
#pragma unroll
    for (int j = 0; j < NB; j += 2) dst[j / 2] = make_double2(d[j], d[j + 1]);
    if (real) {
      double2* dt = reinterpret_cast<double2*>(Dg + lane * ldT);
#pragma unroll
      for (int j = 0; j < NB; j += 2) dt[j / 2] = make_double2(d[j], d[j + 1]);
    }
  }
  __syncwarp();
  const bool up = lane >= 16;
  const int c = lane & 15;
  const double* mp = up ? F + (NB - 1) * LDI + (NB - 1) : F;     // m_ik = mp[sg * (i * LDI + k)]
  const int sg = up ? -1 : 1;
  double x[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) x[i] = (i == (up ? NB - 1 - c : c)) ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    double m[NB];
#pragma unroll
    for (int i = k + 1; i < NB; ++i) m[i] = mp[sg * (i * LDI + k)];
    const double rk = rcs[NB - 1 - k];
    asm volatile("" ::: "memory");   // keep the column's loads here (bounded register pressure)
    if (up) x[k] *= rk;
#pragma unroll
    for (int i = k + 1; i < NB; ++i) x[i] = fma(-m[i], x[k], x[i]);
  }
  __syncwarp();   // all reads of the scratch factors done before U^-1 overwrites it
  double* op = up ? Uinv + (NB - 1) * LDI + c : Linv + c;         // row i of this lane's system -> op[sg * i * LDI]
#pragma unroll
  for (int i = 0; i < NB; ++i) op[sg * i * LDI] = x[i];
  return __any_sync(0xffffffffu, viol);
}

// Pivoting path: inverses of the factored diagonal block already in T (L11\U11 at (jb, jb)), same registers
// scheme as diag_factor without the elimination.
__device__ __forceinline__ void diag_inverses(const double* T, int ldT, int jb, int nb, double* Linv, double* Uinv,
                                              int lane) {
  double d[NB], e[NB], rc[NB];
  const bool mine = lane < nb;
#pragma unroll
  for (int j = 0; j < NB; ++j) d[j] = mine ? T[(jb + lane) * ldT + jb + j] : 0.0;
#pragma unroll
  for (int c = 0; c < NB; ++c) rc[c] = c < nb ? 1.0 / T[(jb + c) * ldT + jb + c] : 0.0;
  // L^-1 by forward substitution on [L | I] (unit diagonal)
#pragma unroll
  for (int j = 0; j < NB; ++j) e[j] = (j == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    if (c < nb) {
      double perow[NB];
#pragma unroll
      for (int j = 0; j <= c; ++j) perow[j] = __shfl_sync(0xffffffffu, e[j], c);
      if (lane > c && mine) {
        const double l = d[c];
#pragma unroll
        for (int j = 0; j <= c; ++j) e[j] = fma(-l, perow[j], e[j]);
      }
    }
  }
  if (lane < NB) {
#pragma unroll
    for (int j = 0; j < NB; ++j) Linv[lane * LDI + j] = mine ? e[j] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) e[j] = (j == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int c = NB - 1; c >= 0; --c) {
    if (c < nb) {
      if (lane == c) {
#pragma unroll
        for (int j = c; j < NB; ++j) e[j] *= rc[c];
      }
      double pf[NB];
#pragma unroll
      for (int j = c; j < NB; ++j) pf[j] = __shfl_sync(0xffffffffu, e[j], c);
      if (lane < c) {
        const double u = d[c];
#pragma unroll
        for (int j = c; j < NB; ++j) e[j] = fma(-u, pf[j], e[j]);
      }
    }
  }
  if (lane < NB) {
#pragma unroll
    for (int j = 0; j < NB; ++j) Uinv[lane * LDI + j] = mine ? e[j] : 0.0;
  }
}

// T[jb..jb+16, c0..c0+8) <- Inv (16x16) * T[jb..jb+16, c0..c0+8), in place; one warp, one column tile. Inv is
// triangular (LOWER: L^-1, else U^-1): the MMAs with its exact-zero 8x8 quadrant are skipped.
template <bool LOWER>
__device__ __forceinline__ void inv_times_tile(double* T, int ldT, int jb, const double* Inv, int c0, int lane) {
  const int gid = lane >> 2, tig = lane & 3, sg = srow(gid);
  double b[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) b[kk] = T[(jb + 4 * kk + tig) * ldT + c0 + gid];
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    if (!LOWER || kk < 2) dmma(acc[0], Inv[sg * LDI + 4 * kk + tig], b[kk]);
    if (LOWER || kk >= 2) dmma(acc[1], Inv[(8 + sg) * LDI + 4 * kk + tig], b[kk]);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
    *reinterpret_cast<double2*>(T + (jb + 8 * i + sg) * ldT + c0 + 2 * tig) = make_double2(acc[i][0], acc[i][1]);
}

__device__ __forceinline__ void backsolve_tile(double* T, int ldT, int ne, const double* Uinv_all, int c0, int lane) {
  const int gid = lane >> 2, tig = lane & 3, sg = srow(gid);
  const int npan = (ne + NB - 1) / NB;
  for (int p = npan - 1; p >= 0; --p) {
    const int jb = p * NB;
    inv_times_tile<false>(T, ldT, jb, Uinv_all + p * NB * LDI, c0, lane);
    __syncwarp();
    if (jb == 0) break;
    const int nk4 = (min(NB, ne - jb) + 3) >> 2;
    double xb[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) xb[kk] = kk < nk4 ? T[(jb + 4 * kk + tig) * ldT + c0 + gid] : 0.0;
    for (int r0 = 0; r0 < jb; r0 += 16) {        // two row tiles per iteration: independent DMMA chains
      double acc[2][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double2 v = *reinterpret_cast<const double2*>(T + (r0 + 8 * i + sg) * ldT + c0 + 2 * tig);
        acc[i][0] = v.x;
        acc[i][1] = v.y;
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (kk < nk4) {
          dmma(acc[0], -T[(r0 + sg) * ldT + jb + 4 * kk + tig], xb[kk]);
          dmma(acc[1], -T[(r0 + 8 + sg) * ldT + jb + 4 * kk + tig], xb[kk]);
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
        *reinterpret_cast<double2*>(T + (r0 + 8 * i + sg) * ldT + c0 + 2 * tig) = make_double2(acc[i][0], acc[i][1]);
    }
    __syncwarp();
  }
}

// T[r0..r0+8, jb..jb+16) <- T[r0..r0+8, jb..jb+16) * Uinv, in place (L21 = A21 U11^-1); one warp, one row tile.
// Returns whether any multiplier exceeds 1 in magnitude (GEPP would have pivoted).
__device__ __forceinline__ bool tile_times_uinv(double* T, int ldT, int jb, const double* Uinv, int r0, int lane) {
  const int gid = lane >> 2, tig = lane & 3, sg = srow(gid);
  double a[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) a[kk] = T[(r0 + sg) * ldT + jb + 4 * kk + tig];
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    if (kk < 2) dmma(acc[0], a[kk], Uinv[(4 * kk + tig) * LDI + gid]);   // U^-1 upper triangular
    dmma(acc[1], a[kk], Uinv[(4 * kk + tig) * LDI + 8 + gid]);
  }
  bool viol = false;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    viol |= fabs(acc[j][0]) > 1.0 || fabs(acc[j][1]) > 1.0;
    *reinterpret_cast<double2*>(T + (r0 + sg) * ldT + jb + 8 * j + 2 * tig) = make_double2(acc[j][0], acc[j][1]);
  }
  return viol;
}

// Pivoting-path panel factorization (GEPP) by one warp directly in T: rows [jb, ne), columns [jb, jb+nb).
// Records piv[k] (absolute row); sets *flag = k+1 at the first exactly-zero pivot.
__device__ __forceinline__ void panel_factor_pivot(double* T, int ldT, int jb, int nb, int ne, int* piv, int* flag,
                                                   int lane) {
  for (int c = 0; c < nb; ++c) {
    const int k = jb + c;
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int r = k + lane; r < ne; r += 32) {
      const double v = fabs(T[r * ldT + k]);
      if (v > best) { best = v; bi = r; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    const int pr = bi < ne ? bi : k;   // all-NaN column (after a zero pivot): keep the row
    if (pr != k && lane < nb) {
      const double t = T[k * ldT + jb + lane];
      T[k * ldT + jb + lane] = T[pr * ldT + jb + lane];
      T[pr * ldT + jb + lane] = t;
    }
    __syncwarp();
    const double pv = T[k * ldT + k];
    const double rp = 1.0 / pv;
    if (lane == 0) {
      piv[k] = pr;
      if ((pv == 0.0 || pv != pv) && *flag == 0) *flag = k + 1;   // zero or NaN pivot (DESIGN R7)
    }
    for (int r = k + 1 + lane; r < ne; r += 32) {
      const double l = T[r * ldT + k] * rp;
      T[r * ldT + k] = l;
      for (int c2 = c + 1; c2 < nb; ++c2) T[r * ldT + jb + c2] = fma(-l, T[k * ldT + jb + c2], T[r * ldT + jb + c2]);
    }
    __syncwarp();
  }
}

// ---- a1 staging with the Tensor Memory Accelerator: bulk row copies global -> shared, completion counted on an
//      mbarrier (transaction bytes), so the next element streams in while the current one computes --------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// shared -> global bulk copy (TMA), tracked by the issuing thread's bulk async-groups
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// wait until every committed bulk group of this thread has finished READING its shared-memory source
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// bulk prefetch of a global range into L2 (TMA engine; no shared memory involved)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// Phase A. PIVOT = false: speculative natural-order pass with look-ahead: while warps 1.. apply the trailing
// update of panel p, warp 0 updates the next 16x16 diagonal block first and factors/inverts it, so the
// sequential diagonal work of panel p+1 overlaps the tensor-core work of panel p. Returns false as soon as GEPP
// would interchange rows (T is then partially overwritten and must be re-staged). PIVOT = true: GEPP, no
// look-ahead.
template <bool PIVOT, int NWARPS>
__device__ __forceinline__ bool phase_a(double* T, const Geo& geo, double* Uinv_all, double* Linv, int* piv,
                                        int* flag, int* spec, int tid, int warp, int lane, uint64_t* mbarB = nullptr,
                                        uint32_t ph = 0, long long* trace = nullptr, int64_t tit = 0) {
  const int ne = geo.ne, R = geo.R8, C8 = geo.C8, ldT = geo.ldT;
  const int npan = (ne + NB - 1) / NB;
  if (!PIVOT && warp == 0) {      // prologue: diagonal block of panel 0 (needs only the A rows)
    if (diag_factor(T, ldT, 0, min(NB, ne), Linv, Uinv_all, lane) && lane == 0) *spec = 1;
  }
  if (mbarB) mbar_wait(mbarB, ph);   // B_e / r_e columns (streamed in during the prologue)
  for (int p = 0; p < npan; ++p) {
    const int jb = p * NB, nb = min(NB, ne - jb);
    double* Uinv = Uinv_all + p * NB * LDI;
    if (PIVOT && warp == 0) {
      panel_factor_pivot(T, ldT, jb, nb, ne, piv, flag, lane);
      __syncwarp();
      diag_inverses(T, ldT, jb, nb, Linv, Uinv, lane);
    }
    __syncthreads();
    HDG_STAMP(trace, tit, 16 + 3 * p);
    if (!PIVOT && *spec) return false;
    if (PIVOT) {   // interchanges of this panel applied to all other columns (thread per column)
      for (int j = tid; j < C8; j += NWARPS * 32) {
        if (j >= jb && j < jb + nb) continue;
        for (int c = 0; c < nb; ++c) {
          const int pr = piv[jb + c];
          if (pr != jb + c) {
            const double t = T[(jb + c) * ldT + j];
            T[(jb + c) * ldT + j] = T[pr * ldT + j];
            T[pr * ldT + j] = t;
          }
        }
      }
      __syncthreads();
    }
    // U12 = L11^-1 A12 (column tiles right of the panel) and, on the fast path, L21 = A21 U11^-1 (row tiles
    // below the panel), distributed over the warps
    const int cj0 = (jb + NB) >> 3, ncj = (C8 >> 3) - cj0;
    const int ri0 = (jb + NB) >> 3, nri = PIVOT ? 0 : (R >> 3) - ri0;
    bool viol = false;
    for (int job = warp; job < ncj + nri; job += NWARPS) {
      if (job < ncj) inv_times_tile<true>(T, ldT, jb, Linv, (cj0 + job) * 8, lane);
      else viol |= tile_times_uinv(T, ldT, jb, Uinv, (ri0 + job - ncj) * 8, lane);
    }
    if (!PIVOT && __any_sync(0xffffffffu, viol) && lane == 0) *spec = 1;
    __syncthreads();
    HDG_STAMP(trace, tit, 17 + 3 * p);
    if (!PIVOT && *spec) return false;
    if (jb + NB < R) {
      const int nk = (nb + 3) & ~3;
      if (PIVOT) {
        mma_update(T, T + jb, T + jb * ldT, ldT, jb + NB, R, jb + NB, C8, nk, warp, NWARPS, lane);
      } else if (warp == 0) {
        // the next diagonal block first (16 x 16), then factor and invert it (look-ahead)
        mma_update(T, T + jb, T + jb * ldT, ldT, jb + NB, jb + 2 * NB, jb + NB, jb + 2 * NB, nk, 0, 1, lane);
        __syncwarp();
        const int jn = jb + NB, nn = min(NB, ne - jn);
        if (diag_factor(T, ldT, jn, nn, Linv, Uinv_all + (p + 1) * NB * LDI, lane) && lane == 0) *spec = 1;
      } else {
        // the rest of the trailing region: rows of the next panel right of its diagonal block, then all rows below
        const int w = warp - 1, nw = NWARPS - 1;
        const int nb_a = (C8 - jb - 2 * NB + 31) >> 5;               // 16x32 blocks in region (a)
        mma_update(T, T + jb, T + jb * ldT, ldT, jb + NB, jb + 2 * NB, jb + 2 * NB, C8, nk, w, nw, lane);
        const int first_b = ((w - nb_a) % nw + nw) % nw;             // continue the round-robin in region (b)
        mma_update(T, T + jb, T + jb * ldT, ldT, jb + 2 * NB, R, jb + NB, C8, nk, first_b, nw, lane);
      }
      HDG_STAMP(trace, tit, 18 + 3 * p);
      if (PIVOT) __syncthreads();
    }
  }
  return true;
}

template <int NWARPS>
__device__ __forceinline__ void stage(double* T, const Geo& geo, const double* A, const double* Bm, const double* re,
                                      const double* sh, int warp, int lane) {
  const int ne = geo.ne, nf = geo.nf, R = geo.R8, CB = geo.CB, C8 = geo.C8, ldT = geo.ldT;
  for (int i = warp; i < R; i += NWARPS) {
    double* Ti = T + i * ldT;
    if (i < ne) {
      const double2* Ai = reinterpret_cast<const double2*>(A + (int64_t)i * ne);
      for (int j = lane; j < ne / 2; j += 32) reinterpret_cast<double2*>(Ti)[j] = __ldg(Ai + j);
      for (int j = ne + lane; j < CB; j += 32) Ti[j] = 0.0;
      const double2* Bi = reinterpret_cast<const double2*>(Bm + (int64_t)i * nf);
      for (int j = lane; j < nf / 2; j += 32) reinterpret_cast<double2*>(Ti + CB)[j] = __ldg(Bi + j);
      if (lane == 0) Ti[CB + nf] = __ldg(re + i);
      for (int j = CB + nf + 1 + lane; j < C8; j += 32) Ti[j] = 0.0;
      if (sh) {   // re-condensation: the diagonal shift of row i
        __syncwarp();
        if (lane == 0) Ti[i] += __ldg(sh + i);
      }
    } else {
      for (int j = lane; j < C8; j += 32) Ti[j] = 0.0;
    }
  }
}

// one warp issues `rows` bulk copies of `bytes` each (row i: src + i*lds -> dst + i*ldd), all counted on bar
__device__ __forceinline__ void issue_rows(double* dst, int ldd, const double* src, int64_t lds, int rows, int cols,
                                           uint64_t* bar, int lane) {
  if (lane == 0) mbar_expect_tx(bar, (uint32_t)rows * (uint32_t)cols * 8u);
  __syncwarp();
  for (int i = lane; i < rows; i += 32) bulk_g2s(dst + i * ldd, src + (int64_t)i * lds, (uint32_t)cols * 8u, bar);
}

constexpr int kChunkCT = 8;   // column tiles of [S | g] per pass of phase B
constexpr int kBatchK = 16;   // k4-steps of C_e fragments loaded ahead in phase B

// Phase B work: NI work items (8-row tile of [S | g] x chunk of kChunkCT column tiles) per warp at a time; all
// their D / r_f / C loads are issued before the first DMMA and the NI independent accumulator sets interleave.
template <int NI, int NWARPS>
__device__ __forceinline__ void schur_items(const SgDst& dst, const double* T, int ldT, int ne, int nf,
                                            int CB, int CTs, int nchunk, const double* Cm, const double* D,
                                            const double* rf, int warp, int lane, bool shareB = false) {
  const int gid = lane >> 2, tig = lane & 3;
  const int nItems = ((nf + 7) >> 3) * nchunk;
  for (int w0 = warp; w0 < nItems; w0 += NI * NWARPS) {
    int row[NI], j0[NI];
    bool rv[NI];
    const double* Crow[NI];
    double acc[NI][kChunkCT][2];
    double cv[NI][kBatchK];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int wi = (w0 + i * NWARPS < nItems) ? w0 + i * NWARPS : w0;
      const int tr = wi / nchunk, ch = wi - tr * nchunk;
      row[i] = tr * 8 + gid;
      rv[i] = (w0 + i * NWARPS < nItems) && row[i] < nf;
      j0[i] = ch * kChunkCT;
      const int rc = rv[i] ? row[i] : 0;
      Crow[i] = Cm + (int64_t)rc * ne;
      const double rfv = __ldg(rf + rc);
#pragma unroll
      for (int j = 0; j < kChunkCT; ++j) {
        const int c = 8 * (j0[i] + j) + 2 * tig;
        const double2 dv = __ldg(reinterpret_cast<const double2*>(D + (int64_t)rc * nf + min(c, nf - 2)));
        const bool on = rv[i] && (j0[i] + j < CTs);
        acc[i][j][0] = on ? (c < nf ? dv.x : (c == nf ? rfv : 0.0)) : 0.0;
        acc[i][j][1] = (on && c < nf) ? dv.y : 0.0;
      }
    }
    for (int k0 = 0; k0 < ne; k0 += 4 * kBatchK) {
      // every load of the batch is issued before any use (no arithmetic on the loaded values here, so they
      // stay in flight together); out-of-range k is clamped, padded rows are zeroed at use
#pragma unroll
      for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int q = 0; q < kBatchK; ++q) cv[i][q] = __ldg(Crow[i] + min(k0 + 4 * q, ne - 4) + tig);
#pragma unroll
      for (int q = 0; q < kBatchK; ++q) {
        const int k = k0 + 4 * q;
        if (k < ne && shareB) {
          // one column chunk (nchunk == 1): the items of a pass share their B fragments — one load per column tile
          const double* Tk = T + (k + tig) * ldT + CB + gid;
          double bf[kChunkCT];
#pragma unroll
          for (int j = 0; j < kChunkCT; ++j) bf[j] = j < CTs ? Tk[8 * j] : 0.0;
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            const double av = rv[i] ? -cv[i][q] : 0.0;
#pragma unroll
            for (int j = 0; j < kChunkCT; ++j)
              if (j < CTs) dmma(acc[i][j], av, bf[j]);
          }
        } else if (k < ne) {
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            const double av = rv[i] ? -cv[i][q] : 0.0;
            const double* Tk = T + (k + tig) * ldT + CB + 8 * j0[i] + gid;
#pragma unroll
            for (int j = 0; j < kChunkCT; ++j)
              if (j0[i] + j < CTs) dmma(acc[i][j], av, Tk[8 * j]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      if (rv[i]) {
#pragma unroll
        for (int j = 0; j < kChunkCT; ++j) {
          const int c = 8 * (j0[i] + j) + 2 * tig;
          if (j0[i] + j < CTs) {
            if (c < nf) out_S2(dst, nf, row[i], c, acc[i][j][0], acc[i][j][1]);
            else if (c == nf) out_g(dst, row[i], acc[i][j][0]);
          }
        }
      }
    }
  }
}

template <int THREADS, int MINB, bool T_SMEM>
__global__ void __launch_bounds__(THREADS, MINB) condense_kernel(const CondenseArgs a) {
  constexpr int NWARPS = THREADS / 32;
  extern __shared__ __align__(16) double smem[];
  const Geo geo(a.ne, a.nf);
  const int ne = geo.ne, nf = geo.nf, CB = geo.CB, C8 = geo.C8, ldT = geo.ldT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int npan = (ne + NB - 1) / NB;
  double* T = T_SMEM ? smem : a.scratch + (int64_t)blockIdx.x * geo.t_doubles();
  double* Uinv_all = T_SMEM ? smem + geo.t_doubles() : smem;
  double* Linv = Uinv_all + npan * NB * LDI;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(Linv + NB * LDI + 48);   // [0]: A rows, [1]: B rows
  int* piv = reinterpret_cast<int*>(mbar + 2);
  int* flag = piv + geo.R8;
  int* spec = flag + 1;

  auto elem_of = [&](int64_t it) -> int64_t { return a.elems ? a.elems[it] : it; };
  // start streaming [A | B] of an element into T; r_e with ordinary loads (one column)
  auto issue_A = [&](int64_t l) { issue_rows(T, ldT, a.A + a.offA[l], ne, ne, ne, &mbar[0], lane); };
  auto issue_B = [&](int64_t l) { issue_rows(T + CB, ldT, a.B + a.offB[l], nf, ne, nf, &mbar[1], lane); };
  auto load_re = [&](int64_t l) {
    for (int i = tid; i < ne; i += THREADS) T[i * ldT + CB + nf] = __ldg(a.re + a.offRe[l] + i);
  };

  if (T_SMEM) {
    // zero T once: the padding rows/columns stay zero through every element (see phase comments)
    for (int i = tid; i < geo.t_doubles(); i += THREADS) T[i] = 0.0;
    if (tid == 0) {
      mbar_init(&mbar[0]);
      mbar_init(&mbar[1]);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (blockIdx.x < a.count) {
      const int64_t l0 = elem_of(blockIdx.x);
      if (warp == 0) {
        issue_A(l0);
        issue_B(l0);
      }
      load_re(l0);
    }
  }
  uint32_t ph = 0;

  for (int64_t it = blockIdx.x; it < a.count; it += gridDim.x, ph ^= 1u) {
    const int64_t l = elem_of(it);
    const double* A = a.A + a.offA[l];
    const double* Bm = a.B + a.offB[l];
    const double* re = a.re + a.offRe[l];
    const int64_t next = it + gridDim.x;

    // ---- a1 stage + a2 (+ forward part of a3) --------------------------------------------------------------
    const double* sh = a.shift ? a.shift + a.offRe[l] : nullptr;
    if (!T_SMEM) stage<NWARPS>(T, geo, A, Bm, re, sh, warp, lane);
    if (tid == 0) { *flag = 0; *spec = 0; }
    const int64_t tit = (it - blockIdx.x) / gridDim.x;
    // phase B reads C_e, D_e, r_f long after they are needed by nothing else: pull them into L2 now
    if (tid == 32) {
      prefetch_l2(a.C + a.offC[l], (uint32_t)(nf * ne * 8));
      prefetch_l2(a.D + a.offD[l], (uint32_t)(nf * nf * 8));
    }
    HDG_STAMP(a.trace, tit, 0);
    if (T_SMEM) {
      mbar_wait(&mbar[0], ph);
      if (sh)
        for (int i = tid; i < ne; i += THREADS) T[i * ldT + i] += __ldg(sh + i);   // before the barrier below
    }
    HDG_STAMP(a.trace, tit, 1);
    __syncthreads();
    HDG_STAMP(a.trace, tit, 2);
    bool pivoted = false;
    if (!phase_a<false, NWARPS>(T, geo, Uinv_all, Linv, piv, flag, spec, tid, warp, lane,
                                T_SMEM ? &mbar[1] : nullptr, ph, a.trace, tit)) {
      pivoted = true;
      __syncthreads();
      stage<NWARPS>(T, geo, A, Bm, re, sh, warp, lane);
      if (tid == 0) { *flag = 0; *spec = 0; }
      __syncthreads();
      phase_a<true, NWARPS>(T, geo, Uinv_all, Linv, piv, flag, spec, tid, warp, lane);
    }
    const int fail = *flag;
    HDG_STAMP(a.trace, tit, 3);

    // ---- a5 factors: L\U row-major + row permutation ---------------------------------------------------------
    {
      double* LU = reinterpret_cast<double*>(a.factors + a.offF[l]);
      // one warp per row, lanes over column pairs: coalesced 16-byte loads and stores, no index division
      // (ne and ldT are even, so every row start is 16-byte aligned in T and in the record)
      // T in shared memory: the rows leave by TMA bulk stores (shared -> global, one per row, asynchronous: the
      // backward substitution and [S | g] never touch T's A columns; warp 0 waits for their shared-memory reads
      // before it streams the next element's A_e in). The warp copy loop cost 5.3 K of C3's 76 K cycles per
      // element (profiles/r02/trace_panel_C3.txt); debug bit 32 keeps it for the A/B.
      const bool bulk = T_SMEM && !fail && !(a.debug & 32);
      if (bulk) {
        fence_proxy_async();   // every thread's writes of T, ordered before the async-proxy reads
        __syncthreads();
        if (warp == 0) {
          for (int i = lane; i < ne; i += 32) bulk_s2g(LU + (size_t)i * ne, T + (size_t)i * ldT, (uint32_t)ne * 8u);
          bulk_commit();
        }
      } else {
        for (int i = warp; i < ne; i += NWARPS) {
          const double2* src = reinterpret_cast<const double2*>(T + (size_t)i * ldT);
          double2* dst = reinterpret_cast<double2*>(LU + (size_t)i * ne);
          for (int j = lane; j < (ne >> 1); j += 32) dst[j] = src[j];
        }
      }
      // row permutation of P A: follow where original row i ends up through the interchanges (parallel in i)
      int32_t* perm = reinterpret_cast<int32_t*>(LU + (int64_t)ne * ne);
      for (int i = tid; i < ne; i += THREADS) {
        int pos = i;
        if (pivoted)
          for (int k = 0; k < ne; ++k) {
            const int pr = piv[k];
            if (pos == k) pos = pr;
            else if (pos == pr) pos = k;
          }
        perm[pos] = i;
      }
      if (tid == 0) a.info[l] = fail;
    }

    if (fail) {
      const double nan = __longlong_as_double(0x7ff8000000000000LL);
      const SgDst dst = sg_dst(a, l);
      for (int i = tid; i < nf * nf; i += THREADS) out_S1(dst, nf, i / nf, i % nf, nan);
      for (int i = tid; i < nf; i += THREADS) out_g(dst, i, nan);
      __syncthreads();
      if (T_SMEM)   // NaNs may have reached the padding: restore the zeros
        for (int i = tid; i < geo.t_doubles(); i += THREADS) T[i] = 0.0;
      __syncthreads();
    } else {
      HDG_STAMP(a.trace, tit, 4);
      // ---- a3 backward part: X = U^-1 W on columns [CB, C8), panels bottom-up ---------------------------------
      for (int ct = warp; ct < ((C8 - CB) >> 3); ct += NWARPS) backsolve_tile(T, ldT, ne, Uinv_all, CB + ct * 8, lane);
      __syncthreads();
      if (a.Xout) {   // §8(f) NEXT #2: the local solutions X = A^-1 [B | r_e] are formed here anyway — save them
        double* Xo = a.Xout + a.offX[l];
        const int nw = nf + 1;
        for (int i = warp; i < ne; i += NWARPS)
          for (int j = lane; j < nw; j += 32) Xo[(int64_t)i * nw + j] = T[i * ldT + CB + j];
      }
    }
    HDG_STAMP(a.trace, tit, 5);
    // the A columns of T are free from here on: start streaming the next element's A_e
    if (T_SMEM && warp == 0) bulk_wait_read_all();   // the factor rows' bulk stores have read T
    if (T_SMEM && warp == 0 && next < a.count) {
      fence_proxy_async();
      issue_A(elem_of(next));
    }

    // ---- a4 Schur complement: [S | g] = [D | r_f] - C X, one warp per 8-row tile, DMMA over k = n_e ----------
    if (!fail) {
      const SgDst dst = sg_dst(a, l);
      const double* Cm = a.C + a.offC[l];
      const double* D = a.D + a.offD[l];
      const double* rf = a.rf + a.offRf[l];
      const int RTs = (nf + 7) >> 3, CTs = (C8 - CB) >> 3;
      const int nchunk = (CTs + kChunkCT - 1) / kChunkCT;
      // One item per warp pass (8 accumulator tiles; more passes) measured faster than two (C3 in one binary:
      // 32.4 vs 33.6 ms; two items sharing their B fragments: 32.8 ms) — debug bit 64 = two items, 128 = shared B
      if (RTs * nchunk > NWARPS && (a.debug & 64))
        schur_items<2, NWARPS>(dst, T, ldT, ne, nf, CB, CTs, nchunk, Cm, D, rf, warp, lane,
                               nchunk == 1 && (a.debug & 128));
      else
        schur_items<1, NWARPS>(dst, T, ldT, ne, nf, CB, CTs, nchunk, Cm, D, rf, warp, lane);
    }
    HDG_STAMP(a.trace, tit, 6);
    __syncthreads();
    HDG_STAMP(a.trace, tit, 7);
    // X has been consumed: stream the next element's B_e and r_e into the right-hand columns
    if (T_SMEM && next < a.count) {
      const int64_t ln = elem_of(next);
      if (warp == 0) {
        fence_proxy_async();
        issue_B(ln);
      }
      load_re(ln);
    }
  }
}

template <int THREADS, int MINB, bool T_SMEM>
cudaError_t launch_t(const CondenseArgs& a, int sms, cudaStream_t s) {
  const Geo geo(a.ne, a.nf);
  const int64_t smem = geo.smem_bytes(T_SMEM);
  auto kern = condense_kernel<THREADS, MINB, T_SMEM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, (size_t)smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = (int64_t)sms * per_sm;
  if (!T_SMEM) grid = sms;   // one scratch slab per resident CTA
  if (grid > a.count) grid = a.count;
  grid = grid_cap(grid);
  kern<<<(unsigned)grid, THREADS, (size_t)smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_condense(const CondenseArgs& a, bool t_in_smem, int sms, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  ++*launches;
  if (!t_in_smem) return launch_t<256, 1, false>(a, sms, s);
  if (a.ne <= 16) return launch_t<64, 6, true>(a, sms, s);
  if (a.ne <= 32) return launch_t<128, 3, true>(a, sms, s);
  if (a.ne <= 64) return launch_t<128, 2, true>(a, sms, s);
  return launch_t<256, 1, true>(a, sms, s);
}

}  // namespace hdg
