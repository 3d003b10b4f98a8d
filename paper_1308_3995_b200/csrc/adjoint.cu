// adjoint.cu — SURVEY.md §8(f) NEXT #1: the adjoint (transposed) use of the condensation path.
// The adjoint local matrix is the transpose of the primal one, so both element-wise steps reuse
// the factors hdg_condense saved (P A_e = L U, row-major L\U + permutation):
//
//     adjoint right-hand side   g~_e = r~_f - B_e^T A_e^-T r~_e         (element part of E~)
//     adjoint reconstruction    u~_e = A_e^-T (r~_e - C_e^T lambda~_e)
//
// with A_e^-T x = P^T L^-T U^-T x: a forward solve with U^T (lower, non-unit), a backward solve with L^T (unit
// upper), then z[perm[i]] = y[i]. One warp per element; the solves in tiles of 8 unknowns: the off-diagonal part
// of each tile is a transposed GEMV on the FP64 tensor cores (DMMA m8n8k4, A fragment = M[k + tig][c0 + gid]:
// eight consecutive doubles of a row per k), the 8x8 diagonal triangle by shuffles. HBM-bound like the primal
// back-substitution (the factors are read once).
#include "dev_common.cuh"
#include "hdg_internal.cuh"

namespace hdg {
namespace {

constexpr int kWarps = 8;

// sum_{k in [k0, k1)} M[k][c0 + i] v[k] for i = lane & 7 (the value lands in lanes 0-7; M row-major with stride ld,
// columns >= ncols and rows >= k1 contribute 0; v zero-padded to a multiple of 4 past k1)
__device__ __forceinline__ double gemv8t(const double* M, int ld, int c0, int ncols, int k0, int k1, const double* v,
                                         int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const bool cv = c0 + gid < ncols;
  double acc0[2] = {0.0, 0.0}, acc1[2] = {0.0, 0.0};
  int k = k0;
#pragma unroll 2
  for (; k + 8 <= k1; k += 8) {
    const double a0 = cv ? __ldg(M + (int64_t)(k + tig) * ld + c0 + gid) : 0.0;
    const double a1 = cv ? __ldg(M + (int64_t)(k + 4 + tig) * ld + c0 + gid) : 0.0;
    const double b0 = gid == 0 ? v[k + tig] : 0.0;
    const double b1 = gid == 0 ? v[k + 4 + tig] : 0.0;
    dmma(acc0, a0, b0);
    dmma(acc1, a1, b1);
  }
  for (; k < k1; k += 4) {
    const bool kv = k + tig < k1;
    const double a0 = (cv && kv) ? __ldg(M + (int64_t)(k + tig) * ld + c0 + gid) : 0.0;
    const double b0 = (gid == 0 && kv) ? v[k + tig] : 0.0;
    dmma(acc0, a0, b0);
  }
  return __shfl_sync(0xffffffffu, acc0[0] + acc1[0], 4 * (lane & 7));
}

// Two column tiles at once: lanes 0-7 get sum_k M[k][c0 + i] v[k] (returned in .x), lanes 0-7 also get
// sum_k M[k][c0 + 8 + i] v[k] (.y): each row contributes 16 consecutive doubles (a whole 128-byte line).
__device__ __forceinline__ double2 gemv16t(const double* M, int ld, int c0, int ncols, int k0, int k1,
                                           const double* v, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const bool cv0 = c0 + gid < ncols, cv1 = c0 + 8 + gid < ncols;
  double accA[2] = {0.0, 0.0}, accB[2] = {0.0, 0.0}, accC[2] = {0.0, 0.0}, accD[2] = {0.0, 0.0};
  int k = k0;
#pragma unroll 2
  for (; k + 8 <= k1; k += 8) {
    const double* r0p = M + (int64_t)(k + tig) * ld + c0 + gid;
    const double* r1p = M + (int64_t)(k + 4 + tig) * ld + c0 + gid;
    const double a0 = cv0 ? __ldg(r0p) : 0.0, a1 = cv1 ? __ldg(r0p + 8) : 0.0;
    const double a2 = cv0 ? __ldg(r1p) : 0.0, a3 = cv1 ? __ldg(r1p + 8) : 0.0;
    const double b0 = gid == 0 ? v[k + tig] : 0.0;
    const double b1 = gid == 0 ? v[k + 4 + tig] : 0.0;
    dmma(accA, a0, b0);
    dmma(accB, a1, b0);
    dmma(accC, a2, b1);
    dmma(accD, a3, b1);
  }
  for (; k < k1; k += 4) {
    const bool kv = k + tig < k1;
    const double* rp = M + (int64_t)(k + tig) * ld + c0 + gid;
    const double a0 = (cv0 && kv) ? __ldg(rp) : 0.0, a1 = (cv1 && kv) ? __ldg(rp + 8) : 0.0;
    const double b0 = (gid == 0 && kv) ? v[k + tig] : 0.0;
    dmma(accA, a0, b0);
    dmma(accB, a1, b0);
  }
  const int src = 4 * (lane & 7);
  return make_double2(__shfl_sync(0xffffffffu, accA[0] + accC[0], src), __shfl_sync(0xffffffffu, accB[0] + accD[0], src));
}

// y = A^-T x in place in vec (length ne), then the permutation into out: out[perm[i]] = y[i]
__device__ __forceinline__ void solve_transposed(const double* LU, const int32_t* perm, int ne, double* vec,
                                                 double* out, int lane) {
  const int nt = (ne + 7) >> 3;
  const int i = lane & 7;
  // U^T v = x (forward): tile T needs U[0 .. r0, r0 .. r0+8) (upper part above the tile) and its 8x8 triangle
  double carry = 0.0;   // tile T's GEMV from the pair pass (odd tiles)
  for (int T = 0; T < nt; ++T) {
    const int r0 = 8 * T, r = r0 + i;
    double s;
    if ((T & 1) == 0) {   // even tile: one pass over rows [0, r0) for this tile and the next
      const double2 s2 = T > 0 ? gemv16t(LU, ne, r0, ne, 0, r0, vec, lane) : make_double2(0.0, 0.0);
      s = s2.x;
      carry = s2.y;
    } else {              // odd tile: the pair pass plus the just-solved rows [r0 - 8, r0)
      s = carry + gemv8t(LU, ne, r0, ne, r0 - 8, r0, vec, lane);
    }
    double Uc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      Uc[j] = (lane < 8 && r < ne && j <= i && r0 + j < ne) ? __ldg(LU + (int64_t)(r0 + j) * ne + r) : 0.0;
    double vi = (lane < 8 && r < ne) ? vec[r] - s : 0.0;
    // the row's reciprocal pivot, off the dependency chain (as in the primal back-substitution)
    double di = 1.0;   // Uc[i] (static selects: a dynamic index would put Uc in local memory)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j == i && lane < 8 && r < ne) di = Uc[j];
    const double rdi = 1.0 / di;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (i == j && lane < 8 && r < ne) vi *= rdi;
      const double vj = __shfl_sync(0xffffffffu, vi, j);
      if (j < i) vi = fma(-Uc[j], vj, vi);
    }
    if (lane < 8 && r < ne) vec[r] = vi;
    __syncwarp();
  }
  // L^T y = v (backward, unit diagonal): tile T needs L[r0+8 .. ne, r0 .. r0+8) (below the tile)
  bool have = false;   // carry holds tile T's GEMV over rows >= r0 + 16 from the pair pass
  for (int T = nt - 1; T >= 0; --T) {
    const int r0 = 8 * T, r = r0 + i, rend = min(r0 + 8, ne);
    double s;
    if (have) {           // second tile of a pair: add the just-solved rows [rend, rend + 8)
      s = carry + gemv8t(LU, ne, r0, ne, rend, min(rend + 8, ne), vec, lane);
      have = false;
    } else if (T > 0) {   // first tile of a pair: one pass over rows [rend, ne) for tiles T - 1 and T
      const double2 s2 = rend < ne ? gemv16t(LU, ne, r0 - 8, ne, rend, ne, vec, lane) : make_double2(0.0, 0.0);
      s = s2.y;
      carry = s2.x;
      have = true;
    } else {
      s = rend < ne ? gemv8t(LU, ne, r0, ne, rend, ne, vec, lane) : 0.0;
    }
    double Lc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      Lc[j] = (lane < 8 && r < ne && j > i && r0 + j < ne) ? __ldg(LU + (int64_t)(r0 + j) * ne + r) : 0.0;
    double yi = (lane < 8 && r < ne) ? vec[r] - s : 0.0;
#pragma unroll
    for (int j = 7; j >= 0; --j) {
      const double yj = __shfl_sync(0xffffffffu, yi, j);
      if (j > i) yi = fma(-Lc[j], yj, yi);
    }
    if (lane < 8 && r < ne) vec[r] = yi;
    __syncwarp();
  }
  for (int k = lane; k < ne; k += 32) out[min((unsigned)__ldg(perm + k), (unsigned)ne - 1)] = vec[k];
  __syncwarp();
}

// MODE 0: g~_e = r~_f - B_e^T A_e^-T r~_e.  MODE 1: u~_e = A_e^-T (r~_e - C_e^T lambda~_e).
template <int MODE>
__global__ void __launch_bounds__(kWarps * 32, 4) adjoint_kernel(const AdjointArgs a) {
  __shared__ double vec_s[kWarps][kMaxNe + 8];
  __shared__ double z_s[kWarps][kMaxNe + 8];
  __shared__ double lam_s[kWarps][kMaxNf + 8];
  const int lane = threadIdx.x & 31;
  const int w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int ne = a.ne, nf = a.nf;
  double* vec = vec_s[w];
  double* z = z_s[w];
  double* lam = lam_s[w];
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  for (int64_t it = (int64_t)blockIdx.x * kWarps + w; it < a.count; it += nwarps) {
    const int64_t l = a.elems ? a.elems[it] : it;
    const double* LU = reinterpret_cast<const double*>(a.factors + a.offF[l]);
    const int32_t* perm = reinterpret_cast<const int32_t*>(LU + (int64_t)ne * ne);
    const double* re = a.re + a.offRe[l];
    if (MODE == 0) {
      for (int k = lane; k < ne + 8; k += 32) vec[k] = k < ne ? __ldg(re + k) : 0.0;
      __syncwarp();
      solve_transposed(LU, perm, ne, vec, z, lane);
      for (int k = ne + lane; k < ne + 8; k += 32) z[k] = 0.0;
      __syncwarp();
      // g~ = r~_f - B^T z, 8 columns of B per tile
      const double* Bm = a.M + a.offM[l];
      double* gt = a.out + a.offOut[l];
      const double* rf = a.rf ? a.rf + a.offRf[l] : nullptr;
      for (int c0 = 0; c0 < nf; c0 += 16) {
        const double2 s = gemv16t(Bm, nf, c0, nf, 0, ne, z, lane);
        const int c = c0 + lane;
        if (lane < 8 && c < nf) gt[c] = (rf ? __ldg(rf + c) : 0.0) - s.x;
        if (lane < 8 && c + 8 < nf) gt[c + 8] = (rf ? __ldg(rf + c + 8) : 0.0) - s.y;
      }
    } else {
      // lambda~_e in slot order (the element's faces, each face's dofs in face_off order), zero padded
      const int64_t e = a.elem_begin + l;
      int f[3], n[3];
#pragma unroll
      for (int s2 = 0; s2 < 3; ++s2) {
        f[s2] = a.elem_face[3 * e + s2];
        n[s2] = f[s2] >= 0 ? a.face_ndof[f[s2]] : 0;
      }
      for (int q = lane; q < nf + 8; q += 32) {
        double v = 0.0;
        if (q < nf) {
          int s2 = 0, qq = q;
          if (qq >= n[0]) { qq -= n[0]; s2 = 1; if (qq >= n[1]) { qq -= n[1]; s2 = 2; } }
          v = __ldg(a.lambda + a.face_off[s2 == 0 ? f[0] : (s2 == 1 ? f[1] : f[2])] + qq);
        }
        lam[q] = v;
      }
      __syncwarp();
      // x = r~_e - C^T lambda~, 8 columns of C per tile
      const double* Cm = a.M + a.offM[l];
      for (int c0 = 0; c0 < ne; c0 += 8) {
        const double s = gemv8t(Cm, ne, c0, ne, 0, nf, lam, lane);
        const int c = c0 + lane;
        if (lane < 8 && c < ne) vec[c] = __ldg(re + c) - s;
      }
      for (int k = ne + lane; k < ne + 8; k += 32) vec[k] = 0.0;
      __syncwarp();
      solve_transposed(LU, perm, ne, vec, a.out + a.offOut[l], lane);
    }
    __syncwarp();
  }
}

template <int MODE>
cudaError_t launch_adj(const AdjointArgs& a, int sms, cudaStream_t s) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adjoint_kernel<MODE>, kWarps * 32, 0);
  if (e != cudaSuccess) return e;
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int64_t need = (a.count + kWarps - 1) / kWarps;
  if (grid > need) grid = need;
  adjoint_kernel<MODE><<<(unsigned)grid, kWarps * 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_adjoint(const AdjointArgs& a, int mode, int sms, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  ++*launches;
  return mode == 0 ? launch_adj<0>(a, sms, s) : launch_adj<1>(a, sms, s);
}

}  // namespace hdg
