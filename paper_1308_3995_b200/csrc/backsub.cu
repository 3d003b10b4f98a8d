// backsub.cu — row a8 of the hot path: element-wise reconstruction after the skeleton solve.
//
//     u_e = A_e^-1 (r_e - B_e lambda_e)          (Eq. ls; "reconstructed inside the elements",
//                                                 PAPER.md:357-359; "reconstruct_local")
// using the factorization saved by hdg_condense: L\U row-major + the row permutation.
//
// HBM-bound streaming kernel, one warp per element. The element's unknowns are processed in tiles of 8 rows. The
// off-diagonal parts — B_e lambda_e, then L_{T,<T} y_{<T} (forward) and U_{T,>T} x_{>T} (backward) — are GEMVs
// on the FP64 tensor cores: DMMA m8n8k4 with the matrix rows as the A fragment (8 rows x 4 columns per load: full
// 32-byte sectors, 8 cache lines per warp instruction instead of the 32 a lane-per-row walk touches) and the
// vector in column 0 of the B fragment (two accumulators interleave the k-steps). The 8x8 diagonal triangle of a
// tile is solved by 8 lanes with shuffles. The solution vector lives in shared memory (one slot per warp).
// Elements with n_e <= 32 use a lane-per-row kernel instead (below).
#include "dev_common.cuh"
#include "hdg_internal.cuh"

namespace hdg {
namespace {

constexpr int kWarps = 8;

// acc (column 0 of an 8x8 accumulator, rows r0 + gid) += M[r0 .. r0+8, k0 .. k1) * v[k0 .. k1); M row-major, ld;
// rows >= nrows and columns >= kv contribute 0 (never read: the last row of a packed array ends at column kv).
// k0, k1 multiples of 4.
__device__ __forceinline__ double gemv8(const double* M, int ld, int r0, int nrows, int k0, int k1, int kv,
                                        const double* v, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const bool rv = r0 + gid < nrows;
  const double* Mr = M + (int64_t)(rv ? r0 + gid : 0) * ld + tig;
  double acc0[2] = {0.0, 0.0}, acc1[2] = {0.0, 0.0};
  int k = k0;
#pragma unroll 4
  for (; k + 8 <= k1; k += 8) {
    const double a0 = (rv && k + tig < kv) ? __ldg(Mr + k) : 0.0;
    const double a1 = (rv && k + 4 + tig < kv) ? __ldg(Mr + k + 4) : 0.0;
    const double b0 = gid == 0 ? v[k + tig] : 0.0;
    const double b1 = gid == 0 ? v[k + 4 + tig] : 0.0;
    dmma(acc0, a0, b0);
    dmma(acc1, a1, b1);
  }
  if (k < k1) {
    const double a0 = (rv && k + tig < kv) ? __ldg(Mr + k) : 0.0;
    const double b0 = gid == 0 ? v[k + tig] : 0.0;
    dmma(acc0, a0, b0);
  }
  // column 0 of the tile sits in lanes with tig == 0 (element 0 of their pair); move row i's value to lane i
  return __shfl_sync(0xffffffffu, acc0[0] + acc1[0], 4 * (lane & 7));
}

// L2 prefetch of rows [r0, r0 + 8) x columns [c0, c1) of the row-major M (one 128-byte line per lane and step):
// the next tile's matrix rows do not depend on the solve, so their HBM latency overlaps the current tile's
__device__ __forceinline__ void prefetch_tile(const double* M, int ld, int r0, int nrows, int c0, int c1, int lane) {
  if (c1 <= c0) return;
  const int lines = (c1 - c0 + 15) >> 4;   // 16 doubles per 128-byte line
  for (int q = lane; q < 8 * lines; q += 32) {
    const int r = r0 + q / lines, c = c0 + 16 * (q % lines);
    if (r < nrows) asm volatile("prefetch.global.L2 [%0];" ::"l"(M + (int64_t)r * ld + c));
  }
}

__global__ void __launch_bounds__(kWarps * 32) backsub_kernel(const BacksubArgs a) {
  __shared__ double vec_s[kWarps][kMaxNe];
  __shared__ double tmp_s[kWarps][kMaxNe];
  __shared__ double lam_s[kWarps][kMaxNf + 4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ne = a.ne, nf = a.nf, nt = (ne + 7) >> 3;
  double* y = vec_s[w];
  double* t = tmp_s[w];
  double* lam = lam_s[w];
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  for (int64_t it = (int64_t)blockIdx.x * kWarps + w; it < a.count; it += nwarps) {
    const int64_t l = a.elems ? a.elems[it] : it;
    const int64_t e = a.elem_begin + l;
    // gather lambda_e in slot order (zero pad to a multiple of 4)
    {
      int f[3], n[3];
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        f[s] = a.elem_face[3 * e + s];
        n[s] = f[s] >= 0 ? a.face_ndof[f[s]] : 0;
      }
      for (int q = lane; q < ((nf + 3) & ~3); q += 32) {
        double v = 0.0;
        if (q < nf) {
          int s = 0, qq = q;
          if (qq >= n[0]) { qq -= n[0]; s = 1; if (qq >= n[1]) { qq -= n[1]; s = 2; } }
          v = __ldg(a.lambda + a.face_off[s == 0 ? f[0] : (s == 1 ? f[1] : f[2])] + qq);
        }
        lam[q] = v;
      }
    }
    __syncwarp();
    const double* Bm = a.B + a.offB[l];
    const double* re = a.re + a.offRe[l];
    const double* LU = reinterpret_cast<const double*>(a.factors + a.offF[l]);
    const int32_t* perm = reinterpret_cast<const int32_t*>(LU + (int64_t)ne * ne);
    // t = r_e - B_e lambda_e (8-row tiles)
    for (int T = 0; T < nt; ++T) {
      const double s = gemv8(Bm, nf, 8 * T, ne, 0, (nf + 3) & ~3, nf, lam, lane);
      const int r = 8 * T + lane;
      if (lane < 8 && r < ne) t[r] = __ldg(re + r) - s;
    }
    __syncwarp();
    // apply P: row i of P t is t[perm[i]]
    for (int i = lane; i < ne; i += 32) y[i] = t[min((unsigned)__ldg(perm + i), (unsigned)ne - 1)];
    __syncwarp();
    // forward: L y = P t (unit lower)
    for (int T = 0; T < nt; ++T) {
      const int r0 = 8 * T;
      if (T + 1 < nt) prefetch_tile(LU, ne, r0 + 8, ne, 0, r0 + 16, lane);
      const double s = T > 0 ? gemv8(LU, ne, r0, ne, 0, r0, ne, y, lane) : 0.0;
      const int i = lane & 7, r = r0 + i;
      double Lr[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) Lr[j] = (lane < 8 && r < ne && j < i) ? __ldg(LU + (int64_t)r * ne + r0 + j) : 0.0;
      double yi = (lane < 8 && r < ne) ? y[r] - s : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double yj = __shfl_sync(0xffffffffu, yi, j);
        if (j < i) yi = fma(-Lr[j], yj, yi);
      }
      if (lane < 8 && r < ne) y[r] = yi;
      __syncwarp();
    }
    // backward: U x = y
    for (int T = nt - 1; T >= 0; --T) {
      const int r0 = 8 * T, rend = min(r0 + 8, ne);
      if (T > 0) prefetch_tile(LU, ne, r0 - 8, ne, r0 - 8, ne, lane);
      const double s = rend < ne ? gemv8(LU, ne, r0, ne, rend, ne, ne, y, lane) : 0.0;
      const int i = lane & 7, r = r0 + i;
      double Ur[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) Ur[j] = (lane < 8 && r < ne && j >= i && r0 + j < ne) ? __ldg(LU + (int64_t)r * ne + r0 + j) : 0.0;
      double xi = (lane < 8 && r < ne) ? y[r] - s : 0.0;
      // the row's reciprocal pivot, off the dependency chain (a division inside it stalled every step and split
      // lanes 0-7 on its slow path)
      const double rdi = (lane < 8 && r < ne) ? 1.0 / __ldg(LU + (int64_t)r * ne + r) : 1.0;
#pragma unroll
      for (int j = 7; j >= 0; --j) {
        if (i == j && lane < 8 && r < ne) xi *= rdi;
        const double xj = __shfl_sync(0xffffffffu, xi, j);
        if (j > i && r0 + j < ne) xi = fma(-Ur[j], xj, xi);
      }
      if (lane < 8 && r < ne) y[r] = xi;
      __syncwarp();
    }
    double* u = a.u + a.offU[l];
    for (int i = lane; i < ne; i += 32) u[i] = y[i];
    __syncwarp();
  }
}

// ---- small elements (n_e <= 32): one lane per row, the whole solve in registers (fewer, longer dependency
//      chains than the tile GEMVs; measured faster for C2: 0.074 vs 0.113 ms) ------------------------------------
constexpr int kWarpsPerBlock = 4;

template <int MAXR>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) backsub_rows_kernel(const BacksubArgs a) {
  __shared__ double lam_s[kWarpsPerBlock][kMaxNf];
  __shared__ double x_s[kWarpsPerBlock][kMaxNe];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ne = a.ne, nf = a.nf;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t it = (int64_t)blockIdx.x * kWarpsPerBlock + w; it < a.count; it += nwarps) {
    const int64_t l = a.elems ? a.elems[it] : it;
    const int64_t e = a.elem_begin + l;
    // gather lambda_e in slot order
    {
      int f[3], n[3];
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        f[s] = a.elem_face[3 * e + s];
        n[s] = f[s] >= 0 ? a.face_ndof[f[s]] : 0;
      }
      for (int q = lane; q < nf; q += 32) {
        int s = 0, qq = q;
        if (qq >= n[0]) { qq -= n[0]; s = 1; if (qq >= n[1]) { qq -= n[1]; s = 2; } }
        lam_s[w][q] = __ldg(a.lambda + a.face_off[s == 0 ? f[0] : (s == 1 ? f[1] : f[2])] + qq);
      }
    }
    __syncwarp();
    const double* Bm = a.B + a.offB[l];
    const double* re = a.re + a.offRe[l];
    const double* LU = reinterpret_cast<const double*>(a.factors + a.offF[l]);
    const int32_t* perm = reinterpret_cast<const int32_t*>(LU + (int64_t)ne * ne);
    double t[MAXR];
    // t = r_e - B_e lambda_e (rows owned by this lane)
#pragma unroll
    for (int s = 0; s < MAXR; ++s) {
      const int i = lane + 32 * s;
      double acc = 0.0;
      if (i < ne) {
        const double2* Bi = reinterpret_cast<const double2*>(Bm + (int64_t)i * nf);
        for (int j = 0; j < nf / 2; ++j) {
          const double2 b = __ldg(Bi + j);
          acc = fma(b.x, lam_s[w][2 * j], acc);
          acc = fma(b.y, lam_s[w][2 * j + 1], acc);
        }
        t[s] = __ldg(re + i) - acc;
        x_s[w][i] = t[s];
      } else {
        t[s] = 0.0;
      }
    }
    __syncwarp();
    // apply P: x_i = t_{perm[i]}
#pragma unroll
    for (int s = 0; s < MAXR; ++s) {
      const int i = lane + 32 * s;
      if (i < ne) t[s] = x_s[w][min((unsigned)__ldg(perm + i), (unsigned)ne - 1)];
    }
    // reciprocals of U's diagonal for the rows this lane owns (off the dependency chain)
    double rd[MAXR];
#pragma unroll
    for (int s = 0; s < MAXR; ++s) {
      const int i = lane + 32 * s;
      rd[s] = i < ne ? 1.0 / __ldg(LU + (int64_t)i * ne + i) : 0.0;
    }
    // forward: L y = P t (unit lower), column k of L = LU[i*ne + k], i > k
#pragma unroll
    for (int s = 0; s < MAXR; ++s) {
      for (int lk = 0; lk < 32; ++lk) {
        const int k = 32 * s + lk;
        if (k >= ne) break;
        const double xk = __shfl_sync(0xffffffffu, t[s], lk);
        const double* Lk = LU + k;
#pragma unroll
        for (int s2 = s; s2 < MAXR; ++s2) {
          const int i = lane + 32 * s2;
          if (i > k && i < ne) t[s2] = fma(-__ldg(Lk + (int64_t)i * ne), xk, t[s2]);
        }
      }
    }
    // backward: U x = y, column k of U = LU[i*ne + k], i < k
#pragma unroll
    for (int s = MAXR - 1; s >= 0; --s) {
      for (int lk = 31; lk >= 0; --lk) {
        const int k = 32 * s + lk;
        if (k >= ne) continue;
        if (lane == lk) t[s] *= rd[s];
        const double xk = __shfl_sync(0xffffffffu, t[s], lk);
        const double* Uk = LU + k;
#pragma unroll
        for (int s2 = 0; s2 <= s; ++s2) {
          const int i = lane + 32 * s2;
          if (i < k) t[s2] = fma(-__ldg(Uk + (int64_t)i * ne), xk, t[s2]);
        }
      }
    }
    double* u = a.u + a.offU[l];
#pragma unroll
    for (int s = 0; s < MAXR; ++s) {
      const int i = lane + 32 * s;
      if (i < ne) u[i] = t[s];
    }
    __syncwarp();
  }
}

template <int MAXR>
cudaError_t launch_rows_t(const BacksubArgs& a, int sms, cudaStream_t s) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, backsub_rows_kernel<MAXR>, kWarpsPerBlock * 32, 0);
  if (e != cudaSuccess) return e;
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int64_t need = (a.count + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (grid > need) grid = need;
  backsub_rows_kernel<MAXR><<<(unsigned)grid, kWarpsPerBlock * 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_backsub(const BacksubArgs& a, int sms, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  ++*launches;
  if (a.ne <= 32) return launch_rows_t<1>(a, sms, s);
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, backsub_kernel, kWarps * 32, 0);
  if (e != cudaSuccess) return e;
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int64_t need = (a.count + kWarps - 1) / kWarps;
  if (grid > need) grid = need;
  backsub_kernel<<<(unsigned)grid, kWarps * 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace hdg
