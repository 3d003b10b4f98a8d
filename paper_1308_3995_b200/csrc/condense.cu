// condense.cu — rows a1-a5 of the hot path: element-local static condensation.
//
// For each element e (Eq. hybridsystem; "condense"):
//     S_e = D_e - C_e A_e^-1 B_e,   g_e = r_f - C_e A_e^-1 r_e,
// with A_e factored by Gaussian elimination with partial pivoting and the factorization kept for
// the reconstruction.
//
// One CTA owns one element at a time (persistent grid). The working matrix T = [A_e | B_e | r_e] lives in
// shared memory (or an L2-resident global scratch slab when it does not fit, hp degrees p >= 4):
//   phase A  : blocked right-looking LU with partial pivoting on the A rows, carried across the B|r columns
//              (T <- [L\U | L^-1 P B | L^-1 P r_e]). Per panel of kNB columns: warp 0 factors the panel
//              (pivot search with warp shuffles, first index on ties like the oracle), all threads apply the
//              row interchanges and the unit-lower triangular solve for U12, then the trailing update
//              T22 -= L21 U12 runs on the FP64 tensor cores (DMMA m8n8k4, operands from shared memory).
//   factors  : L\U written column-major + the row permutation, for the back-substitution kernel.
//   phase A' : blocked backward substitution X = U^-1 [L^-1 P B | L^-1 P r_e] = A_e^-1 [B_e | r_e], in place,
//              trailing updates again on DMMA.
//   phase B  : [S_e | g_e] = [D_e | r_f] - C_e X as one DMMA GEMM per element (n_f x (n_f+1) x n_e), C_e and
//              D_e streamed from HBM straight into the fragments, results stored straight to HBM.
// The flop count equals SURVEY.md §8(d)'s algorithmic count n_e(n_e-1)(4n_e+1)/6 + (n_f+1)(2n_e^2-n_e)
// + 2 n_f n_e (n_f+1) up to O(n_e^2) terms.
#include "hdg_internal.cuh"

namespace hdg {
namespace {

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// dst[r][c] -= sum_{k < nb} As[r][k] * Bs[k][c] over row tiles [r_lo, r_hi) and column tiles [c_lo, c_hi)
// (all multiples of 8; nb multiple of 4). dst, As, Bs share the row stride ld. Work unit: a 2x2 block of 8x8
// tiles per warp, so every A/B fragment loaded from shared memory feeds two DMMAs.
template <int NWARPS>
__device__ __forceinline__ void mma_update(double* dst, const double* As, const double* Bs, int ld, int r_lo, int r_hi,
                                           int c_lo, int c_hi, int nb, int warp, int lane) {
  const int RT = (r_hi - r_lo) >> 3, CT = (c_hi - c_lo) >> 3;
  if (RT <= 0 || CT <= 0) return;
  const int BR = (RT + 1) >> 1, BC = (CT + 1) >> 1;
  const int gid = lane >> 2, tig = lane & 3;
  for (int blk = warp; blk < BR * BC; blk += NWARPS) {
    const int br = blk / BC, bc = blk - br * BC;
    const int r0 = r_lo + br * 16, c0 = c_lo + bc * 16;
    const bool two_r = (br * 2 + 1) < RT, two_c = (bc * 2 + 1) < CT;
    double acc[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if ((i == 0 || two_r) && (j == 0 || two_c)) {
          const double2 v = *reinterpret_cast<const double2*>(dst + (r0 + 8 * i + gid) * ld + c0 + 8 * j + 2 * tig);
          acc[i][j][0] = v.x;
          acc[i][j][1] = v.y;
        } else {
          acc[i][j][0] = 0.0;
          acc[i][j][1] = 0.0;
        }
      }
    for (int k = 0; k < nb; k += 4) {
      const double a0 = -As[(r0 + gid) * ld + k + tig];
      const double a1 = two_r ? -As[(r0 + 8 + gid) * ld + k + tig] : 0.0;
      const double b0 = Bs[(k + tig) * ld + c0 + gid];
      const double b1 = two_c ? Bs[(k + tig) * ld + c0 + 8 + gid] : 0.0;
      dmma(acc[0][0], a0, b0);
      dmma(acc[0][1], a0, b1);
      dmma(acc[1][0], a1, b0);
      dmma(acc[1][1], a1, b1);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if ((i == 0 || two_r) && (j == 0 || two_c))
          *reinterpret_cast<double2*>(dst + (r0 + 8 * i + gid) * ld + c0 + 8 * j + 2 * tig) =
              make_double2(acc[i][j][0], acc[i][j][1]);
  }
}

// Panel factorization by one warp: rows [jb, ne), columns [jb, jb+nb) of T, staged column-major in P.
// Partial pivoting: |pivot| maximal over rows k..ne-1 of the current column, first (lowest) index on ties
// (SURVEY.md §8(c) O1). Records piv[k] (absolute row) and rcp[k] = 1 / pivot; sets *flag = k+1 at the first
// exactly-zero pivot.
__device__ __forceinline__ void panel_factor(double* T, int ldT, double* P, int ldP, int jb, int nb, int ne, int* piv,
                                             double* rcp, int* flag, int lane) {
  const int rows = ne - jb;
  for (int idx = lane; idx < rows * kNB; idx += 32) {
    const int r = idx / kNB, c = idx - r * kNB;
    if (c < nb) P[c * ldP + r] = T[(jb + r) * ldT + jb + c];
  }
  __syncwarp();
  for (int c = 0; c < nb; ++c) {
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int r = c + lane; r < rows; r += 32) {
      const double v = fabs(P[c * ldP + r]);
      if (v > best) { best = v; bi = r; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    const int pr = bi < rows ? bi : c;   // all-NaN column (after a zero pivot): keep the row, stay in range
    if (pr != c && lane < nb) {
      const double t = P[lane * ldP + c];
      P[lane * ldP + c] = P[lane * ldP + pr];
      P[lane * ldP + pr] = t;
    }
    __syncwarp();
    const double pv = P[c * ldP + c];
    const double rp = 1.0 / pv;
    if (lane == 0) {
      piv[jb + c] = jb + pr;
      rcp[jb + c] = rp;
      if (pv == 0.0 && *flag == 0) *flag = jb + c + 1;
    }
    for (int r = c + 1 + lane; r < rows; r += 32) {
      const double l = P[c * ldP + r] * rp;
      P[c * ldP + r] = l;
      for (int c2 = c + 1; c2 < nb; ++c2) P[c2 * ldP + r] -= l * P[c2 * ldP + c];
    }
    __syncwarp();
  }
  for (int idx = lane; idx < rows * kNB; idx += 32) {
    const int r = idx / kNB, c = idx - r * kNB;
    if (c < nb) T[(jb + r) * ldT + jb + c] = P[c * ldP + r];
  }
}

template <int THREADS, bool T_SMEM>
__global__ void __launch_bounds__(THREADS) condense_kernel(const CondenseArgs a) {
  constexpr int NWARPS = THREADS / 32;
  extern __shared__ __align__(16) double smem[];
  const Geo geo(a.ne, a.nf);
  const int ne = geo.ne, nf = geo.nf, R8 = geo.R8, CB = geo.CB, C8 = geo.C8, ldT = geo.ldT, ldP = geo.ldP;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* T = T_SMEM ? smem : a.scratch + (int64_t)blockIdx.x * geo.t_doubles();
  double* P = T_SMEM ? smem + geo.t_doubles() : smem;
  double* rcp = P + kNB * ldP;
  int* piv = reinterpret_cast<int*>(rcp + R8);
  int* flag = piv + R8;
  const int npan = (ne + kNB - 1) / kNB;

  for (int64_t it = blockIdx.x; it < a.count; it += gridDim.x) {
    const int64_t l = a.elems ? a.elems[it] : it;
    const double* A = a.A + a.offA[l];
    const double* Bm = a.B + a.offB[l];
    const double* re = a.re + a.offRe[l];

    // ---- a1 stage: T = [A | 0 | B | r_e | 0], zero rows [ne, R8) -------------------------------------------
    for (int i = warp; i < R8; i += NWARPS) {
      double* Ti = T + i * ldT;
      if (i < ne) {
        const double2* Ai = reinterpret_cast<const double2*>(A + (int64_t)i * ne);
        for (int j = lane; j < ne / 2; j += 32) reinterpret_cast<double2*>(Ti)[j] = __ldg(Ai + j);
        for (int j = ne + lane; j < CB; j += 32) Ti[j] = 0.0;
        const double2* Bi = reinterpret_cast<const double2*>(Bm + (int64_t)i * nf);
        for (int j = lane; j < nf / 2; j += 32) reinterpret_cast<double2*>(Ti + CB)[j] = __ldg(Bi + j);
        if (lane == 0) Ti[CB + nf] = __ldg(re + i);
        for (int j = CB + nf + 1 + lane; j < C8; j += 32) Ti[j] = 0.0;
      } else {
        for (int j = lane; j < C8; j += 32) Ti[j] = 0.0;
      }
    }
    if (tid == 0) *flag = 0;
    __syncthreads();

    // ---- a2 (+ forward part of a3): blocked LU with partial pivoting ---------------------------------------
    for (int p = 0; p < npan; ++p) {
      const int jb = p * kNB, nb = min(kNB, ne - jb);
      if (warp == 0) panel_factor(T, ldT, P, ldP, jb, nb, ne, piv, rcp, flag, lane);
      __syncthreads();
      // row interchanges outside the panel + U12 = L11^-1 A12 (thread per column)
      for (int j = tid; j < C8; j += THREADS) {
        if (j >= jb && j < jb + nb) continue;
        for (int c = 0; c < nb; ++c) {
          const int pr = piv[jb + c];
          if (pr != jb + c) {
            const double t = T[(jb + c) * ldT + j];
            T[(jb + c) * ldT + j] = T[pr * ldT + j];
            T[pr * ldT + j] = t;
          }
        }
        if (j >= jb + nb) {
          double t[kNB];
#pragma unroll
          for (int c = 0; c < kNB; ++c) t[c] = c < nb ? T[(jb + c) * ldT + j] : 0.0;
#pragma unroll
          for (int c = 0; c < kNB; ++c)
#pragma unroll
            for (int c2 = c + 1; c2 < kNB; ++c2)
              if (c2 < nb) t[c2] -= T[(jb + c2) * ldT + jb + c] * t[c];
#pragma unroll
          for (int c = 1; c < kNB; ++c)
            if (c < nb) T[(jb + c) * ldT + j] = t[c];
        }
      }
      __syncthreads();
      if (jb + nb < ne) {
        mma_update<NWARPS>(T, T + jb, T + jb * ldT, ldT, jb + nb, R8, jb + nb, C8, nb, warp, lane);
        __syncthreads();
      }
    }
    const int fail = *flag;

    // ---- a5 factors: L\U column-major + row permutation -----------------------------------------------------
    {
      unsigned char* fb = a.factors + a.offF[l];
      double* LU = reinterpret_cast<double*>(fb);
      // lanes cover a 4 (rows) x 8 (cols) micro-tile: conflict-free smem reads, full 32-byte sector writes
      const int ib = (ne + 3) / 4, kb = (ne + 7) / 8;
      for (int t = warp; t < ib * kb; t += NWARPS) {
        const int i = (t % ib) * 4 + (lane & 3), k = (t / ib) * 8 + (lane >> 2);
        if (k < ne) LU[(int64_t)k * ne + i] = T[i * ldT + k];
      }
      if (tid == 0) {
        int32_t* perm = reinterpret_cast<int32_t*>(LU + (int64_t)ne * ne);
        for (int i = 0; i < ne; ++i) perm[i] = i;
        for (int k = 0; k < ne; ++k) {
          const int pr = piv[k];
          if (pr != k) { const int32_t t = perm[k]; perm[k] = perm[pr]; perm[pr] = t; }
        }
        a.info[l] = fail;
      }
    }

    double* S = a.S + a.offS[l];
    double* g = a.g + a.offG[l];
    if (fail) {
      for (int i = tid; i < nf * nf; i += THREADS) S[i] = __longlong_as_double(0x7ff8000000000000LL);
      for (int i = tid; i < nf; i += THREADS) g[i] = __longlong_as_double(0x7ff8000000000000LL);
      __syncthreads();
      continue;
    }

    // ---- a3 backward part: X = U^-1 W on columns [CB, C8), panels bottom-up -----------------------------------
    for (int p = npan - 1; p >= 0; --p) {
      const int jb = p * kNB, nb = min(kNB, ne - jb);
      for (int j = CB + tid; j < C8; j += THREADS) {
        double t[kNB];
#pragma unroll
        for (int c = 0; c < kNB; ++c) t[c] = c < nb ? T[(jb + c) * ldT + j] : 0.0;
#pragma unroll
        for (int c = kNB - 1; c >= 0; --c) {
          if (c < nb) {
            t[c] *= rcp[jb + c];
#pragma unroll
            for (int c2 = 0; c2 < c; ++c2) t[c2] -= T[(jb + c2) * ldT + jb + c] * t[c];
          }
        }
#pragma unroll
        for (int c = 0; c < kNB; ++c)
          if (c < nb) T[(jb + c) * ldT + j] = t[c];
      }
      __syncthreads();
      if (jb > 0) {
        mma_update<NWARPS>(T, T + jb, T + jb * ldT, ldT, 0, jb, CB, C8, nb, warp, lane);
        __syncthreads();
      }
    }

    // ---- a4 Schur complement: [S | g] = [D | r_f] - C X, one warp per 8-row tile, DMMA over k = n_e ----------
    {
      const double* Cm = a.C + a.offC[l];
      const double* D = a.D + a.offD[l];
      const double* rf = a.rf + a.offRf[l];
      const int RTs = (nf + 7) >> 3, CTs = (C8 - CB) >> 3;
      const int gid = lane >> 2, tig = lane & 3;
      for (int tr = warp; tr < RTs; tr += NWARPS) {
        const int row = tr * 8 + gid;
        const bool rv = row < nf;
        double acc[kMaxCT][2];
#pragma unroll
        for (int j = 0; j < kMaxCT; ++j) {
          const int c = 8 * j + 2 * tig;
          double v0 = 0.0, v1 = 0.0;
          if (j < CTs && rv) {
            if (c < nf) { const double2 d = *reinterpret_cast<const double2*>(D + (int64_t)row * nf + c); v0 = d.x; v1 = d.y; }
            else if (c == nf) v0 = rf[row];
          }
          acc[j][0] = v0;
          acc[j][1] = v1;
        }
        const double* Crow = Cm + (int64_t)(rv ? row : 0) * ne;
#pragma unroll 4
        for (int k = 0; k < ne; k += 4) {
          const double av = rv ? -__ldg(Crow + k + tig) : 0.0;
          const double* Tk = T + (k + tig) * ldT + CB + gid;
#pragma unroll
          for (int j = 0; j < kMaxCT; ++j)
            if (j < CTs) dmma(acc[j], av, Tk[8 * j]);
        }
        if (rv) {
#pragma unroll
          for (int j = 0; j < kMaxCT; ++j) {
            const int c = 8 * j + 2 * tig;
            if (j < CTs) {
              if (c < nf) *reinterpret_cast<double2*>(S + (int64_t)row * nf + c) = make_double2(acc[j][0], acc[j][1]);
              else if (c == nf) g[row] = acc[j][0];
            }
          }
        }
      }
    }
    __syncthreads();
  }
}

template <int THREADS, bool T_SMEM>
cudaError_t launch_t(const CondenseArgs& a, int sms, cudaStream_t s) {
  const Geo geo(a.ne, a.nf);
  const int64_t smem = geo.smem_bytes(T_SMEM);
  cudaError_t e = cudaFuncSetAttribute(condense_kernel<THREADS, T_SMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, condense_kernel<THREADS, T_SMEM>, THREADS, (size_t)smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = (int64_t)sms * per_sm;
  if (!T_SMEM) grid = sms;   // one scratch slab per resident CTA
  if (grid > a.count) grid = a.count;
  condense_kernel<THREADS, T_SMEM><<<(unsigned)grid, THREADS, (size_t)smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_condense(const CondenseArgs& a, bool t_in_smem, int sms, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  ++*launches;
  if (!t_in_smem) return launch_t<256, false>(a, sms, s);
  if (a.ne <= 16) return launch_t<64, true>(a, sms, s);
  if (a.ne <= 32) return launch_t<128, true>(a, sms, s);
  return launch_t<256, true>(a, sms, s);
}

}  // namespace hdg
