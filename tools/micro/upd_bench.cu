// upd_block (condense_sweep.cu's 16x32, k=16 DMMA block update) in isolation: cycles for 1 warp, and the SASS.
#include <cstdio>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int V>
__device__ __noinline__ void upd(double* dst, int ldd, const double* Ap, int lda, const double* Bp, int ldb, int r0, int c0, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double2 v = *reinterpret_cast<const double2*>(dst + (r0 + 8 * i + gid) * ldd + c0 + 8 * j + 2 * tig);
      acc[i][j][0] = v.x; acc[i][j][1] = v.y;
    }
  double a[4][2], b[4][4];
  if (V == 1) {   // all fragments first
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[k][0] = -Ap[(r0 + gid) * lda + 4 * k + tig];
      a[k][1] = -Ap[(r0 + 8 + gid) * lda + 4 * k + tig];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[k][j] = Bp[(4 * k + tig) * ldb + c0 + 8 * j + gid];
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (V == 0) {
      a[k][0] = -Ap[(r0 + gid) * lda + 4 * k + tig];
      a[k][1] = -Ap[(r0 + 8 + gid) * lda + 4 * k + tig];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[k][j] = Bp[(4 * k + tig) * ldb + c0 + 8 * j + gid];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) { dmma(acc[0][j], a[k][0], b[k][j]); dmma(acc[1][j], a[k][1], b[k][j]); }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<double2*>(dst + (r0 + 8 * i + gid) * ldd + c0 + 8 * j + 2 * tig) = make_double2(acc[i][j][0], acc[i][j][1]);
}
template <int V>
__global__ void bench(long long* cyc, int nw) {
  extern __shared__ double T[];
  const int ld = 180, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 120 * ld; i += blockDim.x) T[i] = 0.01 * ((i * 7) % 13);
  __syncthreads();
  long long best = 1LL << 60;
  for (int r = 0; r < 8; ++r) {
    __syncthreads();
    long long t0 = clock64();
    for (int q = 0; q < 8; ++q) upd<V>(T, ld, T + 16, ld, T + 16 * ld, ld, 32 + 16 * ((w + q) % 5), 32 + 32 * (q % 4), lane);
    __syncwarp();
    long long dt = clock64() - t0;
    best = dt < best ? dt : best;
  }
  if (lane == 0) cyc[V * 64 + nw * 8 + w] = best / 8;
}
int main() {
  long long* cyc; cudaMalloc(&cyc, 8 * 256); cudaMemset(cyc, 0, 8 * 256);
  cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 180000);
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 180000);
  for (int nw : {1, 2, 4, 7}) { bench<0><<<1, 32 * nw, 180000>>>(cyc, nw); bench<1><<<1, 32 * nw, 180000>>>(cyc, nw); }
  cudaDeviceSynchronize();
  long long h[256]; cudaMemcpy(h, cyc, 8 * 256, cudaMemcpyDeviceToHost);
  for (int v = 0; v < 2; ++v) for (int nw : {1, 2, 4, 7}) printf("V%d warps %d: %lld cycles per 16x32 block (32 DMMA) per warp -> SM %.1f cyc/DMMA\n", v, nw, h[v * 64 + nw * 8], (double)h[v * 64 + nw * 8] / (32.0 * nw));
}
