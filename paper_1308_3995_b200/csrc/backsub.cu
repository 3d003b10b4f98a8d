// backsub.cu — row a8 of the hot path: element-wise reconstruction after the skeleton solve.
//
//     u_e = A_e^-1 (r_e - B_e lambda_e)          (Eq. ls; "reconstructed inside the elements",
//                                                 PAPER.md:357-359; "reconstruct_local")
// using the factorization saved by hdg_condense: L\U row-major + the row permutation.
//
// HBM-bound streaming kernel, one warp per element, nothing staged in shared memory except lambda_e and the
// permutation buffer: lane i owns rows i, i+32, ... in registers; the triangular solves are column-oriented
// (step k: one shuffle broadcast of x_k, every lane reads element (i, k) of its rows — consecutive k hit the
// same L1 lines of the row-major factor). Many warps per SM hide the n_e-step dependency chain.
#include "hdg_internal.cuh"

namespace hdg {
namespace {

constexpr int kWarpsPerBlock = 4;

template <int MAXR>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) backsub_kernel(const BacksubArgs a) {
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
        lam_s[w][q] = __ldg(a.lambda + a.face_off[f[s]] + qq);
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
      if (i < ne) t[s] = x_s[w][__ldg(perm + i)];
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
cudaError_t launch_t(const BacksubArgs& a, int sms, cudaStream_t s) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, backsub_kernel<MAXR>, kWarpsPerBlock * 32, 0);
  if (e != cudaSuccess) return e;
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int64_t need = (a.count + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (grid > need) grid = need;
  backsub_kernel<MAXR><<<(unsigned)grid, kWarpsPerBlock * 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_backsub(const BacksubArgs& a, int sms, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  ++*launches;
  if (a.ne <= 32) return launch_t<1>(a, sms, s);
  if (a.ne <= 64) return launch_t<2>(a, sms, s);
  if (a.ne <= 128) return launch_t<4>(a, sms, s);
  return launch_t<8>(a, sms, s);
}

}  // namespace hdg
