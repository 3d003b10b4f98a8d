// Latency / throughput of warp primitives on this GPU (one warp), clock64.
#include <cstdio>
__global__ void prims(double* out, long long* cyc, double seed) {
  const int lane = threadIdx.x;
  double x = seed + lane;
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < 256; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) + 1e-9;
  t1 = clock64(); cyc[0] = (t1 - t0) / 256;
  double v[16];
  for (int k = 0; k < 16; ++k) v[k] = x + k;
  t0 = clock64();
  for (int i = 0; i < 32; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __shfl_sync(0xffffffffu, v[k], (lane + k) & 31);
  }
  t1 = clock64(); cyc[1] = (t1 - t0) / (32 * 16);
  for (int k = 0; k < 16; ++k) x += v[k];
  t0 = clock64();
  for (int i = 0; i < 256; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64(); cyc[2] = (t1 - t0) / 256;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) x = 1.0 / (x + 2.0);
  t1 = clock64(); cyc[3] = (t1 - t0) / 64;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) {
    const double y = x + 2.0;
    double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
    double e = fma(-y, r, 1.0); r = fma(r, e, r); e = fma(-y, r, 1.0); x = fma(r, e, r);
  }
  t1 = clock64(); cyc[4] = (t1 - t0) / 64;
  __shared__ double s[64];
  s[lane] = x; s[lane + 32] = x;
  __syncwarp();
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < 256; ++i) { double w = s[idx]; idx = (int)(w * 0.0) + ((idx + 1) & 31); x += w; }
  t1 = clock64(); cyc[5] = (t1 - t0) / 256;
  out[lane] = x;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 256); cudaMalloc(&cyc, 64);
  prims<<<1, 32>>>(out, cyc, 0.5);
  prims<<<1, 32>>>(out, cyc, 0.5);
  long long h[8]; cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
  printf("shfl.f64 dependent latency %lld | shfl.f64 independent interval %lld | dfma latency %lld | div latency %lld | rcp+2newton latency %lld | lds chain %lld\n", h[0], h[1], h[2], h[3], h[4], h[5]);
}
