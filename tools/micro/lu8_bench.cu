// condense_sweep.cu's lu8 timed alone (hot loop) in a small kernel, vs the same call inside a loop that also runs
// the chain's other per-panel code — isolating the in-kernel slowdown of the diagonal factorization.
#include "../../paper_1308_3995_b200/csrc/condense_sweep.cu"
#include <cstdio>
namespace hdg { namespace {
__global__ void bench(double* LUg, long long* cyc) {
  __shared__ __align__(16) double T[16 * 20], T0[16 * 20], Li[16 * LDI], Ui[16 * LDI], St[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < 320; i += 32) T0[i] = ((i % 20) == (i / 20)) ? 4.0 + 0.1 * (i / 20) : 0.01 * ((i * 7) % 11) - 0.05;
  __syncwarp();
  long long best = 1LL << 60, first = 0;
  bool v = false;
  for (int r = 0; r < 20; ++r) {
    for (int i = lane; i < 320; i += 32) T[i] = T0[i];
    __syncwarp();
    long long t0 = clock64();
    v |= lu8(T, 20, 0, 8, Li, Ui, LUg, 16, St, lane);
    long long dt = clock64() - t0;
    best = dt < best ? dt : best;
    if (r == 0) first = dt;
  }
  if (lane == 0) { cyc[0] = best; cyc[1] = first; cyc[2] = v; }
}
}}
int main() {
  double* LUg; long long* cyc; cudaMalloc(&LUg, 256 * 8); cudaMalloc(&cyc, 64);
  hdg::bench<<<1, 32>>>(LUg, cyc); cudaDeviceSynchronize();
  long long h[3]; cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
  printf("lu8 alone: best %lld first %lld cycles (viol %lld)\n", h[0], h[1], h[2]);
}
