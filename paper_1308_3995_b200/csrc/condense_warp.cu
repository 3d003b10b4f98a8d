// condense_warp.cu — rows a1-a5 of the hot path for small elements (n_e <= 32, n_f + 1 <= 64):
// one WARP per element, many elements in flight per SM (C1: n_e = 12, C2: n_e = 24). For these sizes the per-element
// dependency chain (n_e pivot steps) — not bandwidth or FP64 throughput — bounds a CTA-per-element kernel, so the
// latency is hidden by running 8 elements per CTA and several CTAs per SM.
//
//     S_e = D_e - C_e A_e^-1 B_e,   g_e = r_f - C_e A_e^-1 r_e        (Eq. hybridsystem)
//
// Lane i holds row i of [A_e | B_e | r_e] in registers. Gaussian elimination with partial pivoting
// as in SURVEY.md §8(c) O1, done without moving rows: each lane tracks the position its row occupies in GEPP's
// interchanged order; step k picks, among the rows at positions >= k, the largest |a_ik| (lowest position on
// ties: exactly GEPP's strict-'>' scan), the pivot row is broadcast through shared memory, and every row below
// takes its multiplier (a true division by the pivot, as the oracle) and updates [A | B r] — so the row operations
// are bit-for-bit those of GEPP on physically swapped rows. Then X = U^-1 W (W = L^-1 P [B r]) by backward column
// sweeps, X goes to shared memory, and [S | g] = [D | r_f] - C_e X on the FP64 tensor cores (DMMA m8n8k4, C_e
// fragments straight from global, D_e / r_f as the accumulator). Factors: L\U rows written in GEPP order
// (row-major) + the permutation, the layout hdg_backsubstitute reads.
#include "dev_common.cuh"
#include "hdg_internal.cuh"

namespace hdg {
namespace {

constexpr int kWarpsPerCta = 8;

template <int NE, int NW>   // NE >= n_e (registers per row of A), NW >= n_f + 1 (registers per row of [B r])
__global__ void __launch_bounds__(kWarpsPerCta * 32) warp_kernel(const CondenseArgs a) {
  constexpr int LDX = NW + 4 - (NW % 16 == 12 ? 8 : 0);   // X row stride (doubles)
  extern __shared__ __align__(16) double wsm[];             // per warp: pivot row [NE + NW] | X [32 x LDX]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int ne = a.ne, nf = a.nf, nw = nf + 1;
  double* prow = wsm + (size_t)w * (NE + NW + 32 * LDX);
  double* X = prow + NE + NW;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerCta;
  for (int64_t it = (int64_t)blockIdx.x * kWarpsPerCta + w; it < a.count; it += nwarps) {
    const int64_t l = a.elems ? a.elems[it] : it;
    const double* A = a.A + a.offA[l];
    const double* Bm = a.B + a.offB[l];
    const double* re = a.re + a.offRe[l];
    const bool real = lane < ne;
    double d[NE], wv[NW];
#pragma unroll
    for (int j = 0; j < NE; ++j) d[j] = (real && j < ne) ? __ldg(A + (int64_t)lane * ne + j) : 0.0;
#pragma unroll
    for (int j = 0; j < NW; ++j)
      wv[j] = real ? (j < nf ? __ldg(Bm + (int64_t)lane * nf + j) : (j == nf ? __ldg(re + lane) : 0.0)) : 0.0;
    int pos = real ? lane : 1 << 20;   // position of this lane's row in GEPP's interchanged order
    int fail = 0;
    // ---- GEPP on [A | B r] -----------------------------------------------------------------------------------
#pragma unroll
    for (int k = 0; k < NE; ++k) {
      if (k < ne) {
        // pivot search among rows at positions >= k: max |a_ik|, ties -> lowest position
        double best = (pos >= k && pos < (1 << 20)) ? fabs(d[k]) : -1.0;
        int bpos = pos >= k ? pos : (1 << 30);
        int blane = lane;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, off);
          const int op = __shfl_xor_sync(0xffffffffu, bpos, off);
          const int ol = __shfl_xor_sync(0xffffffffu, blane, off);
          if (ob > best || (ob == best && op < bpos)) { best = ob; bpos = op; blane = ol; }
        }
        // the row at position k swaps places with the pivot row
        const int kl = __ballot_sync(0xffffffffu, pos == k) ? __ffs(__ballot_sync(0xffffffffu, pos == k)) - 1 : 0;
        const int ppos = __shfl_sync(0xffffffffu, pos, blane);
        if (lane == kl) pos = ppos;
        if (lane == blane) pos = k;
        // broadcast the pivot row (columns > k of A, all of [B r])
        if (lane == blane) {
#pragma unroll
          for (int j = 0; j < NE; ++j)
            if (j >= k) prow[j] = d[j];
#pragma unroll
          for (int j = 0; j < NW; ++j) prow[NE + j] = wv[j];
        }
        __syncwarp();
        const double pv = prow[k];
        if (pv == 0.0 || !(pv == pv)) fail = fail ? fail : k + 1;
        if (pos > k && pos < (1 << 20) && pv != 0.0) {
          const double m = d[k] / pv;   // a true division, as the oracle
          d[k] = m;
#pragma unroll
          for (int j = 0; j < NE; ++j)
            if (j > k) d[j] = fma(-m, prow[j], d[j]);
#pragma unroll
          for (int j = 0; j < NW; ++j) wv[j] = fma(-m, prow[NE + j], wv[j]);
        }
        __syncwarp();
      }
    }
    // ---- factors: row i of P A (the row at position i) + permutation ---------------------------------------------
    double* LU = reinterpret_cast<double*>(a.factors + a.offF[l]);
    int32_t* perm = reinterpret_cast<int32_t*>(LU + (int64_t)ne * ne);
    if (real) {
#pragma unroll
      for (int j = 0; j < NE; ++j)
        if (j < ne) LU[(int64_t)pos * ne + j] = d[j];
      perm[pos] = lane;
    }
    if (lane == 0) a.info[l] = fail;
    double* S = a.S + a.offS[l];
    double* g = a.g + a.offG[l];
    if (fail) {
      for (int i = lane; i < nf * nf; i += 32) S[i] = __longlong_as_double(0x7ff8000000000000LL);
      for (int i = lane; i < nf; i += 32) g[i] = __longlong_as_double(0x7ff8000000000000LL);
      __syncwarp();
      continue;
    }
    // ---- X = U^-1 W: backward column sweeps over positions ne-1 .. 0 -------------------------------------------
#pragma unroll
    for (int k = NE - 1; k >= 0; --k) {
      if (k < ne) {
        if (pos == k) {
          const double rd = 1.0 / d[k];
#pragma unroll
          for (int j = 0; j < NW; ++j) {
            wv[j] *= rd;
            prow[NE + j] = wv[j];
          }
        }
        __syncwarp();
        if (pos < k) {
          const double u = d[k];
#pragma unroll
          for (int j = 0; j < NW; ++j) wv[j] = fma(-u, prow[NE + j], wv[j]);
        }
        __syncwarp();
      }
    }
    // X rows by position (= unknown index of A_e^-1 [B r])
    if (real) {
#pragma unroll
      for (int j = 0; j < NW; ++j) X[pos * LDX + j] = wv[j];
    }
    __syncwarp();
    // ---- [S | g] = [D | r_f] - C X on DMMA: 8 x 8 tiles, k over n_e --------------------------------------------
    const double* Cm = a.C + a.offC[l];
    const double* D = a.D + a.offD[l];
    const double* rf = a.rf + a.offRf[l];
    const int RT = (nf + 7) >> 3, CT = (nw + 7) >> 3;
    for (int t = 0; t < RT * CT; ++t) {
      const int rt = t / CT, ct = t - rt * CT;
      const int row = rt * 8 + gid, c = ct * 8 + 2 * tig;
      double acc[2];
      acc[0] = row < nf ? (c < nf ? __ldg(D + (int64_t)row * nf + c) : (c == nf ? __ldg(rf + row) : 0.0)) : 0.0;
      acc[1] = (row < nf && c + 1 < nf) ? __ldg(D + (int64_t)row * nf + c + 1) : 0.0;
      const int crow = rt * 8 + gid;
#pragma unroll
      for (int k = 0; k < NE; k += 4) {
        if (k < ne) {
          const double av = (crow < nf && k + tig < ne) ? -__ldg(Cm + (int64_t)crow * ne + k + tig) : 0.0;
          const double bv = (k + tig < ne) ? X[(k + tig) * LDX + ct * 8 + gid] : 0.0;
          dmma(acc, av, bv);
        }
      }
      if (row < nf) {
        if (c < nf) *reinterpret_cast<double2*>(S + (int64_t)row * nf + c) = make_double2(acc[0], acc[1]);
        else if (c == nf) g[row] = acc[0];
      }
    }
    __syncwarp();
  }
}

template <int NE, int NW>
cudaError_t launch_w(const CondenseArgs& a, int sms, cudaStream_t s) {
  constexpr int LDX = NW + 4 - (NW % 16 == 12 ? 8 : 0);
  const size_t smem = sizeof(double) * kWarpsPerCta * (NE + NW + 32 * LDX);
  cudaError_t e = cudaFuncSetAttribute(warp_kernel<NE, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, warp_kernel<NE, NW>, kWarpsPerCta * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = (int64_t)sms * per_sm;
  const int64_t need = (a.count + kWarpsPerCta - 1) / kWarpsPerCta;
  if (grid > need) grid = need;
  warp_kernel<NE, NW><<<(unsigned)grid, kWarpsPerCta * 32, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool warp_supported(int ne, int nf) { return ne <= 32 && nf + 1 <= 64; }

cudaError_t launch_condense_warp(const CondenseArgs& a, int sms, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  ++*launches;
  const int nw = a.nf + 1;
  if (a.ne <= 12 && nw <= 32) return launch_w<12, 32>(a, sms, s);
  if (a.ne <= 16 && nw <= 40) return launch_w<16, 40>(a, sms, s);
  if (a.ne <= 24 && nw <= 40) return launch_w<24, 40>(a, sms, s);
  if (a.ne <= 32 && nw <= 40) return launch_w<32, 40>(a, sms, s);
  return launch_w<32, 64>(a, sms, s);
}

}  // namespace hdg
