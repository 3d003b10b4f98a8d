// condense_warp.cu — rows a1-a5 of the hot path for small elements (n_e <= 32,
// n_e + n_f + 1 <= 64): one WARP per element, no CTA barriers, 16 elements in flight per SM (C1: n_e = 12,
// C2: n_e = 24). At these sizes the per-element dependency chain — not bandwidth or FP64 throughput — bounds a
// CTA-per-element kernel; here independent warps hide it.
//
//     S_e = D_e - C_e A_e^-1 B_e,   g_e = r_f - C_e A_e^-1 r_e        (Eq. hybridsystem)
//
// The warp holds T = [A_e | B_e | r_e] in its slice of shared memory (row-major) and runs Gaussian elimination
// with partial pivoting on it exactly as the oracle does (largest |a_ik|, lowest
// row on ties, true division for the multipliers, rows interchanged), which turns T into [L\U | L^-1 P [B r]];
// then X = U^-1 W column by column (each lane owns columns), and [S | g] = [D | r_f] - C_e X on the FP64 tensor
// cores (DMMA m8n8k4: C_e fragments from global, X fragments from shared memory, D_e / r_f as the accumulator).
// Compact loops over shared memory, not register arrays: a fully unrolled register-resident elimination measured
// ~40 % of its stall samples on instruction fetch (C2: 0.97 ms vs this kernel's number in DESIGN §11).
// Factors: L\U row-major in GEPP row order + the permutation (the layout hdg_backsubstitute reads).
#include "dev_common.cuh"
#include "hdg_internal.cuh"

namespace hdg {
namespace {

constexpr int kWarpsPerCta = 4;
constexpr int kLdT = 65;       // row stride of T (>= 64 columns; odd: row-wise (lane = column) and column-wise
                               // (lane = row) accesses both conflict-free)
constexpr int kMaxTiles = 5;   // 8-wide column tiles of [S | g] (n_f + 1 <= 40)

template <int NE, bool FUSED>
__global__ void __launch_bounds__(kWarpsPerCta * 32, 4) warp_kernel(const CondenseArgs a) {
  extern __shared__ __align__(16) double wsm[];
  const int lane = threadIdx.x & 31;
  const int w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int gid = lane >> 2, tig = lane & 3;
  const int ne = a.ne, nf = a.nf, nw = nf + 1, nc = ne + nw;
  double* T = wsm + (size_t)w * NE * kLdT;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerCta;
  const int c0 = lane, c1 = lane + 32;   // this lane's columns of T
  // element l's A_e into T's columns [0, ne) by asynchronous 8-byte copies (no registers, no wait here)
  auto copy_A = [&](int64_t l_) {
    if (lane < ne) {
      const double* A_ = a.A + a.offA[l_];
      for (int i = 0; i < ne; ++i)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(T + i * kLdT + lane)),
                     "l"(A_ + (int64_t)i * ne + lane) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  bool pref = false;   // this element's A_e already in flight (issued during the previous element's [S | g] tiles)
  for (int64_t it = (int64_t)blockIdx.x * kWarpsPerCta + w; it < a.count; it += nwarps) {
    const int64_t l = a.elems ? a.elems[it] : it;
    // no L2 prefetch: measured on C2, the next element's blocks prefetched at this element's start 0.673 ms (ncu:
    // 22 % L2 hit rate, 1.76x the algorithmic DRAM reads — an element's run time ahead, the lines were evicted
    // before use), a short-distance schedule (this element's C_e, D_e at its start, the next A_e, B_e before the
    // [S | g] tiles) 0.639 ms, none 0.629 ms (C1 0.0399 / 0.0418 / 0.0397 ms). Instead the next element's A_e is
    // copied straight into T's dead A columns while this element's [S | g] tiles run.
    if (!pref) copy_A(l);
    pref = false;
    const double* Bm = a.B + a.offB[l];
    const double* re = a.re + a.offRe[l];
    const double* sh = a.shift ? a.shift + a.offRe[l] : nullptr;   // re-condensation: A_e + diag(shift_e)
    // ---- W = [B_e | r_e] into T's columns [ne, nc) by asynchronous 8-byte copies: they land while the
    //      elimination of A_e runs (the row interchanges and L^-1 reach W only after it) ---------------------------
    {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = h ? c1 : c0;
        if (c >= ne && c < nc) {
          const bool isr = c == ne + nf;
          for (int i = 0; i < ne; ++i)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(T + i * kLdT + c)),
                         "l"(isr ? re + i : Bm + (int64_t)i * nf + (c - ne)) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");   // A_e has landed (this lane's copies; W may not)
    if (sh && lane < ne) T[lane * kLdT + lane] += __ldg(sh + lane);   // re-condensation: A_e + diag(shift_e)
    int prow = lane;   // original row now at position `lane`
    int fail = 0;
    __syncwarp();
    // 8x8-tile DMMA update of T: rows [r0, r0 + 8) (< rlim), columns [cb, cb + 8) (< clim)
    //   T[rows][cols] -= T[rows][kc .. kc + nk) * T[kr .. kr + nk)[cols]        (nk a multiple of 4, <= 8)
    auto tile_update = [&](int r0, int rlim, int cb, int clim, int kc, int kr, int nk) {
      const int row = r0 + gid, col = cb + 2 * tig;
      const bool rv = row < rlim;
      double acc[2];
      acc[0] = (rv && col < clim) ? T[row * kLdT + col] : 0.0;
      acc[1] = (rv && col + 1 < clim) ? T[row * kLdT + col + 1] : 0.0;
      const bool bv = cb + gid < clim;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        if (4 * kk < nk) {
          const double av = rv ? -T[row * kLdT + kc + 4 * kk + tig] : 0.0;
          const double bw = bv ? T[(kr + 4 * kk + tig) * kLdT + cb + gid] : 0.0;
          dmma(acc, av, bw);
        }
      }
      if (rv && col < clim) T[row * kLdT + col] = acc[0];
      if (rv && col + 1 < clim) T[row * kLdT + col + 1] = acc[1];
    };
    // one panel of a unit-lower block solve: rows [k0, k0 + nb) <- L11^-1 rows (lane = column, L11 by broadcast), then
    // rows [k0 + nb, ne) -= L21 * those rows on 8x8 DMMA tiles (k = nb); columns [cb, ce)
    auto lower_panel = [&](int k0, int nb, int cb, int ce) {
      {   // columns cb + lane and cb + lane + 32 together: one broadcast load of L11 feeds both
        const int ca = cb + lane, cc = cb + lane + 32;
        const bool h0 = ca < ce, h1 = cc < ce;
        double t[8], v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          t[r] = (h0 && r < nb) ? T[(k0 + r) * kLdT + ca] : 0.0;
          v[r] = (h1 && r < nb) ? T[(k0 + r) * kLdT + cc] : 0.0;
        }
#pragma unroll
        for (int r = 1; r < 8; ++r) {
          if (r < nb) {
#pragma unroll
            for (int q = 0; q < r; ++q) {
              const double lq = T[(k0 + r) * kLdT + k0 + q];
              t[r] = fma(-lq, t[q], t[r]);
              v[r] = fma(-lq, v[q], v[r]);
            }
            if (h0) T[(k0 + r) * kLdT + ca] = t[r];
            if (h1) T[(k0 + r) * kLdT + cc] = v[r];
          }
        }
      }
      __syncwarp();
      const int ke = k0 + nb;
      if (ke < ne && cb < ce) {
        const int ntc = (ce - cb + 7) >> 3, ntile = ((ne - ke + 7) >> 3) * ntc;
        for (int q = 0; q < ntile; ++q) tile_update(ke + (q / ntc) * 8, ne, cb + (q % ntc) * 8, ce, k0, k0, nb);
        __syncwarp();
      }
    };
    // ---- GEPP on T, blocked by 8 columns (right-looking): inside a panel each step is the oracle's — pivot = max
    //      |a_ik| over positions i >= k with the lowest position on ties, whole rows interchanged, true division for
    //      the multipliers — with the rank-1 update restricted to the panel's columns (lane = row); then U12 =
    //      L11^-1 A12 on the panel rows (lane = column) and A22 -= L21 U12 on the FP64 tensor cores. Every pivot
    //      column is fully updated before its search, so this is GEPP, not a speculation; only the rounding order
    //      of the trailing sums differs from the oracle's one-step-at-a-time updates ------------------------------
    for (int k0 = 0; k0 < ne && !fail; k0 += 8) {
      const int nb = min(8, ne - k0), ke = k0 + nb;
      for (int k = k0; k < ke; ++k) {
        // pivot: max |a_ik| over positions i >= k, lowest position on ties (the oracle's strict '>' scan): the
        // maximum by a butterfly, then the lowest candidate lane holding it by a ballot (NaNs never win; all-NaN
        // candidates leave the pivot in place and fail below)
        const double mag = (lane >= k && lane < ne) ? fabs(T[lane * kLdT + k]) : -1.0;
        double best = mag;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
        const unsigned hit = __ballot_sync(0xffffffffu, lane >= k && lane < ne && mag == best);
        const int p = hit ? __ffs(hit) - 1 : k;
        if (p != k) {   // warp-uniform
          if (c0 < ne) {   // A's columns only: W takes the final permutation after the elimination
            double* rk = T + k * kLdT;
            double* rq = T + p * kLdT;
            const double t0 = rk[c0], q0 = rq[c0];
            rk[c0] = q0;
            rq[c0] = t0;
          }
          const int pk = __shfl_sync(0xffffffffu, prow, k), pp = __shfl_sync(0xffffffffu, prow, p);
          if (lane == k) prow = pp;
          if (lane == p) prow = pk;
        }
        __syncwarp();
        const double piv = T[k * kLdT + k];
        if (piv == 0.0 || !(piv == piv)) {   // warp-uniform
          fail = k + 1;
          break;
        }
        const bool mine = lane > k && lane < ne;
        double li = 0.0;
        if (mine) {
          li = T[lane * kLdT + k] / piv;   // multipliers (true division, as the oracle)
          T[lane * kLdT + k] = li;
        }
        for (int j = k + 1; j < ke; ++j) {   // the panel's columns only (lane = row)
          const double u = T[k * kLdT + j];
          if (mine) T[lane * kLdT + j] = fma(-li, u, T[lane * kLdT + j]);
        }
        __syncwarp();
      }
      if (fail) break;
      lower_panel(k0, nb, ke, ne);   // U12 = L11^-1 A12, A22 -= L21 U12 over A's columns
    }
    // ---- factors: L\U rows in GEPP order (row-major, coalesced per row) + the permutation — also for a singular
    //      element (its partial factors; prow is a permutation however far the elimination got), so the factor
    //      record always holds a valid permutation for the solve kernels ---------------------------------------------
    double* LU = reinterpret_cast<double*>(a.factors + a.offF[l]);
    int32_t* perm = reinterpret_cast<int32_t*>(LU + (int64_t)ne * ne);
    for (int i = 0; i < ne; ++i)
      if (c0 < ne) LU[(int64_t)i * ne + c0] = T[i * kLdT + c0];
    if (lane < ne) perm[lane] = prow;
    if (lane == 0) a.info[l] = fail;
    if (fail) {
      const double nan = __longlong_as_double(0x7ff8000000000000LL);
      const SgDst dst = sg_dst(a, l);
      for (int i = lane; i < nf * nf; i += 32) out_S1(dst, nf, i / nf, i % nf, nan);
      for (int i = lane; i < nf; i += 32) out_g(dst, i, nan);
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");   // W's copies must land before T is reused
      __syncwarp();
      continue;
    }
    // ---- W <- L^-1 P W: W's copies have landed; rows into GEPP order (position i <- original row prow[i]), then
    //      the unit-lower solve panel by panel -----------------------------------------------------------------------
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = h ? c1 : c0;
      const bool act = c >= ne && c < nc;
      double v[NE];
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        const int src = __shfl_sync(0xffffffffu, prow, i);
        v[i] = (act && i < ne) ? T[src * kLdT + c] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < NE; ++i)
        if (act && i < ne) T[i * kLdT + c] = v[i];
    }
    __syncwarp();
    for (int k0 = 0; k0 < ne; k0 += 8) lower_panel(k0, min(8, ne - k0), ne, nc);
    // ---- [S | g] row-tile operands, one tile ahead: C_e fragments (negated) and the D_e / r_f accumulators; the
    //      first tile's loads are issued here and land during the triangular solve --------------------------------
    const double* Cm = a.C + a.offC[l];
    const double* D = a.D + a.offD[l];
    const double* rf = a.rf + a.offRf[l];
    const int RT = (nf + 7) >> 3, CT = (nw + 7) >> 3;
    auto load_rt = [&](int rt, double (&af)[NE / 4], double (&accs)[kMaxTiles][2]) {
      const int row = rt * 8 + gid;
      const bool rv = rt < RT && row < nf;
#pragma unroll
      for (int kk = 0; kk < NE / 4; ++kk)
        af[kk] = (rv && 4 * kk + tig < ne) ? -__ldg(Cm + (int64_t)row * ne + 4 * kk + tig) : 0.0;
#pragma unroll
      for (int ct = 0; ct < kMaxTiles; ++ct) {
        const int c = ct * 8 + 2 * tig;
        const bool tv = rv && ct < CT;
        accs[ct][0] = tv ? (c < nf ? __ldg(D + (int64_t)row * nf + c) : (c == nf ? __ldg(rf + row) : 0.0)) : 0.0;
        accs[ct][1] = tv ? (c + 1 < nf ? __ldg(D + (int64_t)row * nf + c + 1) : (c + 1 == nf ? __ldg(rf + row) : 0.0)) : 0.0;
      }
    };
    double af[NE / 4], accs[kMaxTiles][2];
    load_rt(0, af, accs);
    // ---- X = U^-1 W, blocked by 8 rows from the bottom: the diagonal 8x8 triangle per W column (lane = column, one
    //      reciprocal per pivot: the back-solve decides nothing), then the rows above -= U12 X_b on DMMA tiles ------
    {
      const bool a0 = c0 >= ne && c0 < nc, a1 = c1 < nc;
      for (int r0 = (ne - 1) & ~7; r0 >= 0; r0 -= 8) {
        const int nr = min(8, ne - r0);
        const double rdl = lane < nr ? 1.0 / T[(r0 + lane) * kLdT + r0 + lane] : 0.0;   // one reciprocal per lane
        double rd[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) rd[r] = __shfl_sync(0xffffffffu, rdl, r);
        {   // this lane's W columns c0 (if >= ne) and c1 together: one broadcast load of U feeds both
          const bool h0 = c0 >= ne && c0 < nc, h1 = c1 < nc;
          double t[8], v[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            t[r] = (h0 && r < nr) ? T[(r0 + r) * kLdT + c0] : 0.0;
            v[r] = (h1 && r < nr) ? T[(r0 + r) * kLdT + c1] : 0.0;
          }
#pragma unroll
          for (int r = 7; r >= 0; --r) {
            if (r < nr) {
#pragma unroll
              for (int q = r + 1; q < 8; ++q) {
                if (q < nr) {
                  const double u = T[(r0 + r) * kLdT + r0 + q];
                  t[r] = fma(-u, t[q], t[r]);
                  v[r] = fma(-u, v[q], v[r]);
                }
              }
              t[r] *= rd[r];
              v[r] *= rd[r];
              if (h0) T[(r0 + r) * kLdT + c0] = t[r];
              if (h1) T[(r0 + r) * kLdT + c1] = v[r];
            }
          }
        }
        __syncwarp();
        if (r0 > 0) {
          const int ntc = (nw + 7) >> 3, ntile = (r0 >> 3) * ntc;
          for (int q = 0; q < ntile; ++q) tile_update((q / ntc) * 8, r0, ne + (q % ntc) * 8, nc, r0, r0, nr);
          __syncwarp();
        }
      }
      __syncwarp();   // every read of T's A columns (U) is done
      if (it + nwarps < a.count) {
        copy_A(a.elems ? a.elems[it + nwarps] : it + nwarps);
        pref = true;
      }
      if (a.Xout) {   // §8(f) NEXT #2: the local solutions X = A^-1 [B | r_e] (columns ne .. nc of T) — save them
        __syncwarp();
        double* Xo = a.Xout + a.offX[l];
        for (int i = 0; i < ne; ++i) {
          if (a0) Xo[(int64_t)i * nw + c0 - ne] = T[i * kLdT + c0];
          if (a1) Xo[(int64_t)i * nw + c1 - ne] = T[i * kLdT + c1];
        }
      }
      // W's padding columns [nc, kLdT) read as zeros by the last X fragment
      if (c0 >= nc)
        for (int i = 0; i < ne; ++i) T[i * kLdT + c0] = 0.0;
      if (c1 >= nc && c1 < kLdT)
        for (int i = 0; i < ne; ++i) T[i * kLdT + c1] = 0.0;
    }
    __syncwarp();
    // ---- [S | g] = [D | r_f] - C X on DMMA: 8 x 8 tiles, k over n_e (X = columns ne.. of T) --------------------------
    const SgDst dst = FUSED ? sg_dst(a, l) : SgDst{};
    const double* X = T + ne;
    for (int rt = 0; rt < RT; ++rt) {
      const int row = rt * 8 + gid;
      const bool rv = row < nf;
      double afn[NE / 4], accn[kMaxTiles][2];
      load_rt(rt + 1, afn, accn);   // the next row tile's operands while this one runs (zeros past the last)
#pragma unroll
      for (int ct = 0; ct < kMaxTiles; ++ct) {
        if (ct >= CT) break;
        const int c = ct * 8 + 2 * tig;
        double (&acc)[2] = accs[ct];
#pragma unroll
        for (int kk = 0; kk < NE / 4; ++kk)
          if (4 * kk < ne) dmma(acc, af[kk], (4 * kk + tig < ne) ? X[(4 * kk + tig) * kLdT + ct * 8 + gid] : 0.0);
        if (rv) {
          if constexpr (FUSED) {   // hdg_condense_assemble: straight into K, E
            if (c + 1 < nf) {
              out_S2(dst, nf, row, c, acc[0], acc[1]);
            } else if (c + 1 == nf) {   // odd n_f: the pair straddles S's last column and g
              out_S1(dst, nf, row, c, acc[0]);
              out_g(dst, row, acc[1]);
            } else if (c == nf) {
              out_g(dst, row, acc[0]);
            }
          } else {
            double* S = a.S + a.offS[l];
            double* g = a.g + a.offG[l];
            if (c + 1 < nf) {
              *reinterpret_cast<double2*>(S + (int64_t)row * nf + c) = make_double2(acc[0], acc[1]);
            } else if (c + 1 == nf) {
              S[(int64_t)row * nf + c] = acc[0];
              g[row] = acc[1];
            } else if (c == nf) {
              g[row] = acc[0];
            }
          }
        }
      }
#pragma unroll
      for (int kk = 0; kk < NE / 4; ++kk) af[kk] = afn[kk];
#pragma unroll
      for (int ct = 0; ct < kMaxTiles; ++ct) {
        accs[ct][0] = accn[ct][0];
        accs[ct][1] = accn[ct][1];
      }
    }
    __syncwarp();
  }
}

template <int NE>
cudaError_t launch_w(const CondenseArgs& a, int sms, cudaStream_t s) {
  const size_t smem = sizeof(double) * kWarpsPerCta * NE * kLdT;
  auto kern = a.Kf ? warp_kernel<NE, true> : warp_kernel<NE, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarpsPerCta * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = (int64_t)sms * per_sm;
  const int64_t need = (a.count + kWarpsPerCta - 1) / kWarpsPerCta;
  if (grid > need) grid = need;
  grid = grid_cap(grid);
  kern<<<(unsigned)grid, kWarpsPerCta * 32, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

// n_e <= 32 (one row per lane in the pivot search), n_e + n_f + 1 <= 64 (two columns of T per lane), n_f + 1 <= 40
// (column tiles of [S | g]), even n_f and n_e a multiple of 4 (whole DMMA k-steps; 16-byte prefetch sizes)
bool warp_supported(int ne, int nf) {
  return ne <= 32 && ne % 4 == 0 && nf % 2 == 0 && ne + nf + 1 <= 64 && nf + 1 <= 8 * kMaxTiles;
}

cudaError_t launch_condense_warp(const CondenseArgs& a, int sms, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  ++*launches;
  if (a.ne <= 12) return launch_w<12>(a, sms, s);
  if (a.ne <= 16) return launch_w<16>(a, sms, s);
  if (a.ne <= 24) return launch_w<24>(a, sms, s);
  return launch_w<32>(a, sms, s);
}

}  // namespace hdg
