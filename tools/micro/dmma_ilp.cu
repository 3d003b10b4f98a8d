// Per-warp DMMA issue rate vs independent accumulator chains (ILP), operands in distinct registers, 1..8 warps.
#include <cstdio>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int N>
__global__ void k(double* out, long long* cyc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc[N][2], a[N], b[N];
#pragma unroll
  for (int i = 0; i < N; ++i) { acc[i][0] = acc[i][1] = 0; a[i] = 1e-3 * (lane + i); b[i] = 1e-3 * (i + 1); }
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < 64; ++r) {
#pragma unroll
    for (int i = 0; i < N; ++i) dmma(acc[i], a[i], b[(i + r) % N]);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) s += acc[i][0] + acc[i][1];
  out[threadIdx.x] = s;
  if (lane == 0) cyc[w] = (t1 - t0);
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8 * 64);
  long long h[64];
  auto run = [&](auto kern, int n, int nw) {
    kern<<<1, 32 * nw>>>(out, cyc); kern<<<1, 32 * nw>>>(out, cyc); cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8 * 64, cudaMemcpyDeviceToHost);
    printf("chains %2d warps %2d: %.1f cycles per DMMA per warp, SM %.2f cyc/DMMA\n", n, nw, h[0] / (64.0 * n), h[0] / (64.0 * n * nw));
  };
  for (int nw : {1, 2, 4, 8, 16}) { run(k<1>, 1, nw); run(k<4>, 4, nw); run(k<8>, 8, nw); run(k<16>, 16, nw); }
}
