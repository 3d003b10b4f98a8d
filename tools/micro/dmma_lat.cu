// DMMA m8n8k4 latency (dependent chain) and per-warp issue interval (independent accumulators), alone and with
// a second DMMA-streaming warp on the same SMSP (warp 4 of the CTA) — calibration for the sweep kernel.
#include <cstdio>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__global__ void k(double* out, long long* cyc, int other) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  double a = 1.0 + 1e-3 * lane, b = 0.999;
  if (warp == 0) {
    double acc[8][2] = {};
    long long t0 = clock64();
    for (int i = 0; i < 64; ++i) dmma(acc[0], a, b);
    long long t1 = clock64();
    for (int i = 0; i < 16; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(acc[j], a, b);
    }
    long long t2 = clock64();
    double x = acc[0][0];
    for (int i = 0; i < 64; ++i) x = fma(x, 0.999, 1e-3);
    long long t3 = clock64();
    double y = x;
    for (int i = 0; i < 64; ++i) y = __shfl_sync(0xffffffffu, y, (lane + 1) & 31) * 1.0000001;
    long long t4 = clock64();
    double v[16];
    for (int j = 0; j < 16; ++j) v[j] = y + j;
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __shfl_sync(0xffffffffu, v[j], (lane + j) & 31);
    long long t5 = clock64();
    if (lane == 0) {
      cyc[other * 8 + 0] = (t1 - t0) / 64;
      cyc[other * 8 + 1] = (t2 - t1) / 128;
      cyc[other * 8 + 2] = (t3 - t2) / 64;
      cyc[other * 8 + 3] = (t4 - t3) / 64;
      cyc[other * 8 + 4] = (t5 - t4) / 128;
      done = 1;
    }
    double s = 0; for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1];
    for (int j = 0; j < 16; ++j) s += v[j];
    out[lane] = s + x + y;
  } else if (warp == 4 && other) {
    double acc[4][2] = {};
    while (!done) {
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(acc[j], a, b);
    }
    out[64 + lane] = acc[0][0] + acc[1][0] + acc[2][0] + acc[3][0];
  }
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1024); cudaMalloc(&cyc, 256);
  for (int o = 0; o < 2; ++o) { k<<<1, 256>>>(out, cyc, o); k<<<1, 256>>>(out, cyc, o); cudaDeviceSynchronize(); }
  long long h[16]; cudaMemcpy(h, cyc, 128, cudaMemcpyDeviceToHost);
  for (int o = 0; o < 2; ++o)
    printf("%s: dmma dep latency %lld | dmma indep interval %lld | dfma dep latency %lld | shfl.f64 dep latency %lld | shfl.f64 indep interval %lld\n",
           o ? "with DMMA warp on same SMSP" : "alone", h[o*8], h[o*8+1], h[o*8+2], h[o*8+3], h[o*8+4]);
}
