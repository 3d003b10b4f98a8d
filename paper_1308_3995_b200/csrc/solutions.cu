// solutions.cu — SURVEY.md §8(f) NEXT #2: the saved local solutions ("the solutions to Eq. (ls) can
// be saved after the assembly of the hybridized system and reused during the reconstruction").
//
//   save:     X_e = A_e^-1 [B_e | r_e]   (n_e x (n_f + 1), row-major; the last column is y_e = A_e^-1 r_e)
//   reuse:    u_e = y_e - X_e[:, 0:n_f] lambda_e   (= A_e^-1 (r_e - B_e lambda_e), Eq. ls)
//
// save_kernel: one element per CTA at a time (persistent grid), the right-hand sides R = P [B_e | r_e] staged in
// shared memory; each warp owns 8-column tiles of R and runs the forward (unit L) and backward (U) substitutions on
// them in 8-row tiles: the off-diagonal parts are FP64 tensor-core MMAs (m8n8k4, the factor rows as A fragments —
// 32-byte sector reads from the factor record — and the solved row tiles of R as B fragments, two accumulator
// chains), the 8x8 diagonal triangles by shuffles. X leaves with coalesced stores.
// backsub_saved_kernel: one warp per element; lambda_e gathered in slot order, the GEMV on DMMA (X rows as A
// fragments, lambda in column 0 of B), u = y - s. HBM-bound: n_e (n_f + 1) doubles read per element.
#include <algorithm>

#include "dev_common.cuh"
#include "hdg_internal.cuh"

namespace hdg {
namespace {

constexpr int kSaveWarps = 8;

__global__ void __launch_bounds__(kSaveWarps * 32) save_kernel(const SolutionsArgs a) {
  extern __shared__ __align__(16) double R[];
  const int ne = a.ne, nf = a.nf, nw = nf + 1;
  const int RA = round_up(ne, 8), NT = RA / 8, CW = round_up(nw, 8), CT = CW / 8;
  const int ldR = pad_ld(CW);
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int gid = lane >> 2, tig = lane & 3;
  for (int64_t it = blockIdx.x; it < a.count; it += gridDim.x) {
    const int64_t l = a.elems ? a.elems[it] : it;
    const double* LU = reinterpret_cast<const double*>(a.factors + a.offF[l]);
    const int32_t* perm = reinterpret_cast<const int32_t*>(LU + (int64_t)ne * ne);
    const double* Bm = a.B + a.offB[l];
    const double* re = a.re + a.offRe[l];
    // ---- R = P [B | r_e] (row i of P A is row perm[i] of A), zero padding rows / columns
    for (int i = warp; i < RA; i += kSaveWarps) {
      const int src = i < ne ? min((unsigned)__ldg(perm + i), (unsigned)ne - 1) : 0;
      for (int j = lane; j < CW; j += 32) {
        double v = 0.0;
        if (i < ne) v = j < nf ? __ldg(Bm + (int64_t)src * nf + j) : (j == nf ? __ldg(re + src) : 0.0);
        R[i * ldR + j] = v;
      }
    }
    __syncthreads();
    for (int ct = warp; ct < CT; ct += kSaveWarps) {
      const int c0 = 8 * ct;
      // ---- forward: L Y = P [B r] (unit lower), row tile by row tile
      for (int T = 0; T < NT; ++T) {
        const int row = 8 * T + gid;
        const bool rv = row < ne;
        const double* Lr = LU + (int64_t)(rv ? row : 0) * ne;
        double acc0[2], acc1[2] = {0.0, 0.0}, acc2[2] = {0.0, 0.0}, acc3[2] = {0.0, 0.0};
        {
          const double2 v = *reinterpret_cast<const double2*>(R + row * ldR + c0 + 2 * tig);
          acc0[0] = v.x;
          acc0[1] = v.y;
        }
        // two row tiles per iteration, all four factor loads issued before the MMAs (four accumulator chains):
        // the L2 latency of the factor rows is paid once per two tiles, not per MMA
        int k = 0;
        for (; k + 2 <= T; k += 2) {
          const int kc = 8 * k + tig;
          const double a0 = rv ? -__ldg(Lr + kc) : 0.0, a1 = rv ? -__ldg(Lr + kc + 4) : 0.0;
          const double a2 = rv ? -__ldg(Lr + kc + 8) : 0.0, a3 = rv ? -__ldg(Lr + kc + 12) : 0.0;
          dmma(acc0, a0, R[kc * ldR + c0 + gid]);
          dmma(acc1, a1, R[(kc + 4) * ldR + c0 + gid]);
          dmma(acc2, a2, R[(kc + 8) * ldR + c0 + gid]);
          dmma(acc3, a3, R[(kc + 12) * ldR + c0 + gid]);
        }
        if (k < T) {
          const int kc = 8 * k + tig;
          const double a0 = rv ? -__ldg(Lr + kc) : 0.0, a1 = rv ? -__ldg(Lr + kc + 4) : 0.0;
          dmma(acc0, a0, R[kc * ldR + c0 + gid]);
          dmma(acc1, a1, R[(kc + 4) * ldR + c0 + gid]);
        }
        acc0[0] += acc1[0] + (acc2[0] + acc3[0]);
        acc0[1] += acc1[1] + (acc2[1] + acc3[1]);
        double Lrow[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) Lrow[r] = (rv && 8 * T + r < ne && r < gid) ? __ldg(Lr + 8 * T + r) : 0.0;
#pragma unroll
        for (int r = 0; r < 7; ++r) {
          const double v0 = __shfl_sync(0xffffffffu, acc0[0], 4 * r + tig);
          const double v1 = __shfl_sync(0xffffffffu, acc0[1], 4 * r + tig);
          if (gid > r) {
            acc0[0] = fma(-Lrow[r], v0, acc0[0]);
            acc0[1] = fma(-Lrow[r], v1, acc0[1]);
          }
        }
        *reinterpret_cast<double2*>(R + row * ldR + c0 + 2 * tig) = make_double2(acc0[0], acc0[1]);
        __syncwarp();
      }
      // ---- backward: U X = Y
      for (int T = NT - 1; T >= 0; --T) {
        const int row = 8 * T + gid;
        const bool rv = row < ne;
        const double* Ur = LU + (int64_t)(rv ? row : 0) * ne;
        double acc0[2], acc1[2] = {0.0, 0.0}, acc2[2] = {0.0, 0.0}, acc3[2] = {0.0, 0.0};
        {
          const double2 v = *reinterpret_cast<const double2*>(R + row * ldR + c0 + 2 * tig);
          acc0[0] = v.x;
          acc0[1] = v.y;
        }
        int k = T + 1;
        for (; k + 2 <= NT; k += 2) {
          const int kc = 8 * k + tig;
          const double a0 = (rv && kc < ne) ? -__ldg(Ur + kc) : 0.0, a1 = (rv && kc + 4 < ne) ? -__ldg(Ur + kc + 4) : 0.0;
          const double a2 = (rv && kc + 8 < ne) ? -__ldg(Ur + kc + 8) : 0.0;
          const double a3 = (rv && kc + 12 < ne) ? -__ldg(Ur + kc + 12) : 0.0;
          dmma(acc0, a0, R[kc * ldR + c0 + gid]);
          dmma(acc1, a1, R[(kc + 4) * ldR + c0 + gid]);
          dmma(acc2, a2, R[(kc + 8) * ldR + c0 + gid]);
          dmma(acc3, a3, R[(kc + 12) * ldR + c0 + gid]);
        }
        if (k < NT) {
          const int kc = 8 * k + tig;
          const double a0 = (rv && kc < ne) ? -__ldg(Ur + kc) : 0.0, a1 = (rv && kc + 4 < ne) ? -__ldg(Ur + kc + 4) : 0.0;
          dmma(acc0, a0, R[kc * ldR + c0 + gid]);
          dmma(acc1, a1, R[(kc + 4) * ldR + c0 + gid]);
        }
        acc0[0] += acc1[0] + (acc2[0] + acc3[0]);
        acc0[1] += acc1[1] + (acc2[1] + acc3[1]);
        double Urow[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) Urow[r] = (rv && 8 * T + r < ne && r > gid) ? __ldg(Ur + 8 * T + r) : 0.0;
        const double rdiag = rv ? 1.0 / __ldg(Ur + row) : 1.0;   // padding rows: unit diagonal
#pragma unroll
        for (int r = 7; r >= 0; --r) {
          if (gid == r) {
            acc0[0] *= rdiag;
            acc0[1] *= rdiag;
          }
          const double v0 = __shfl_sync(0xffffffffu, acc0[0], 4 * r + tig);
          const double v1 = __shfl_sync(0xffffffffu, acc0[1], 4 * r + tig);
          if (gid < r) {
            acc0[0] = fma(-Urow[r], v0, acc0[0]);
            acc0[1] = fma(-Urow[r], v1, acc0[1]);
          }
        }
        *reinterpret_cast<double2*>(R + row * ldR + c0 + 2 * tig) = make_double2(acc0[0], acc0[1]);
        __syncwarp();
      }
    }
    __syncthreads();
    // ---- X_e (n_e x (n_f + 1), contiguous): coalesced stores
    double* X = a.X + a.offX[l];
    for (int q = tid; q < ne * nw; q += kSaveWarps * 32) {
      const int i = q / nw, j = q - i * nw;
      X[q] = R[i * ldR + j];
    }
    __syncthreads();
  }
}

constexpr int kBsWarps = 8;

__global__ void __launch_bounds__(kBsWarps * 32) backsub_saved_kernel(const SolutionsArgs a) {
  __shared__ double lam_s[kBsWarps][kMaxNf + 8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int ne = a.ne, nf = a.nf, nw = nf + 1, nt = (ne + 7) >> 3, nk = (nf + 3) & ~3;
  double* lam = lam_s[w];
  const int64_t nwarps = (int64_t)gridDim.x * kBsWarps;
  for (int64_t it = (int64_t)blockIdx.x * kBsWarps + w; it < a.count; it += nwarps) {
    const int64_t l = a.elems ? a.elems[it] : it;
    const int64_t e = a.elem_begin + l;
    {
      int f[3], n[3];
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        f[s] = a.elem_face[3 * e + s];
        n[s] = f[s] >= 0 ? a.face_ndof[f[s]] : 0;
      }
      for (int q = lane; q < nk; q += 32) {
        double v = 0.0;
        if (q < nf) {
          int s = 0, qq = q;
          if (qq >= n[0]) { qq -= n[0]; s = 1; if (qq >= n[1]) { qq -= n[1]; s = 2; } }
          v = __ldg(a.lambda + a.face_off[f[s]] + qq);
        }
        lam[q] = v;
      }
    }
    __syncwarp();
    const double* X = a.Xin + a.offX[l];
    double* u = a.u + a.offU[l];
    for (int T = 0; T < nt; ++T) {
      const int row = 8 * T + gid;
      const bool rv = row < ne;
      const double* Xr = X + (int64_t)(rv ? row : 0) * nw;
      double acc0[2] = {0.0, 0.0}, acc1[2] = {0.0, 0.0};
      int k = 0;
#pragma unroll 2
      for (; k + 8 <= nk; k += 8) {
        const double a0 = (rv && k + tig < nf) ? __ldg(Xr + k + tig) : 0.0;
        const double a1 = (rv && k + 4 + tig < nf) ? __ldg(Xr + k + 4 + tig) : 0.0;
        dmma(acc0, a0, gid == 0 ? lam[k + tig] : 0.0);
        dmma(acc1, a1, gid == 0 ? lam[k + 4 + tig] : 0.0);
      }
      if (k < nk) {
        const double a0 = (rv && k + tig < nf) ? __ldg(Xr + k + tig) : 0.0;
        dmma(acc0, a0, gid == 0 ? lam[k + tig] : 0.0);
      }
      // column 0 of the tile sits in lanes with tig == 0; row i's sum to lane i
      const double s = __shfl_sync(0xffffffffu, acc0[0] + acc1[0], 4 * (lane & 7));
      const int r = 8 * T + lane;
      if (lane < 8 && r < ne) u[r] = __ldg(X + (int64_t)r * nw + nf) - s;
    }
    __syncwarp();
  }
}

}  // namespace

cudaError_t launch_save_solutions(const SolutionsArgs& a, int sms, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  ++*launches;
  const int RA = round_up(a.ne, 8), ldR = pad_ld(round_up(a.nf + 1, 8));
  const size_t smem = sizeof(double) * (size_t)RA * ldR;
  cudaError_t e = cudaFuncSetAttribute(save_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, save_kernel, kSaveWarps * 32, smem);
  if (e != cudaSuccess) return e;
  int64_t grid = (int64_t)sms * std::max(per_sm, 1);
  if (grid > a.count) grid = a.count;
  save_kernel<<<(unsigned)grid, kSaveWarps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_backsub_saved(const SolutionsArgs& a, int sms, cudaStream_t s, int64_t* launches) {
  if (a.count <= 0) return cudaSuccess;
  ++*launches;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, backsub_saved_kernel, kBsWarps * 32, 0);
  if (e != cudaSuccess) return e;
  int64_t grid = (int64_t)sms * std::max(per_sm, 1);
  const int64_t need = (a.count + kBsWarps - 1) / kBsWarps;
  if (grid > need) grid = need;
  backsub_saved_kernel<<<(unsigned)grid, kBsWarps * 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace hdg
