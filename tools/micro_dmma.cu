#include <cstdio>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double acc[NACC][2];
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < 256; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i], a, b);
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 256;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  long long h;
  k<1><<<1, 32>>>(out, cyc, 1e-3, 1e-3); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("1 acc chain: %lld cycles per DMMA (latency)\n", h);
  k<2><<<1, 32>>>(out, cyc, 1e-3, 1e-3); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("2 acc: %lld cycles per round\n", h);
  k<4><<<1, 32>>>(out, cyc, 1e-3, 1e-3); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("4 acc: %lld cycles per round\n", h);
  k<8><<<1, 32>>>(out, cyc, 1e-3, 1e-3); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("8 acc: %lld cycles per round\n", h);
  k<8><<<1, 64>>>(out, cyc, 1e-3, 1e-3); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("8 acc, 2 warps (2 SMSPs): %lld cycles per round\n", h);
  k<8><<<1, 160>>>(out, cyc, 1e-3, 1e-3); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("8 acc, 5 warps: %lld cycles per round\n", h);
}
