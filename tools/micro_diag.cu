// Microbenchmark: latency of the condensation kernel's device building blocks, one warp, clock64.
#include "../paper_1308_3995_b200/csrc/condense.cu"
#include <cstdio>

namespace hdg { namespace {
__global__ void bench_diag(double* out, long long* cyc, int reps, int which) {
  __shared__ double T[16 * 20 + 64], T0[16 * 20 + 64];
  __shared__ double Linv[16 * 20], Uinv[16 * 20], buf[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < 16 * 20; i += 32) T0[i] = (i % 21 == 0) ? 4.0 : 0.01 * (i % 7);
  __syncwarp();
  long long t0 = 0;
  bool v = false;
  long long acc = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = lane; i < 16 * 20; i += 32) T[i] = T0[i];
    __syncwarp();
    t0 = clock64();
    if (which == 0) v |= diag_factor(T, 20, 0, 16, Linv, Uinv, buf, lane);
    else if (which == 1) diag_inverses(T, 20, 0, 16, Linv, Uinv, lane);
    else if (which == 2) inv_times_tile(T, 20, 0, Linv, 0, lane);
    __syncwarp();
    acc += clock64() - t0;
  }
  if (lane == 0) { cyc[which] = acc / reps; out[0] = T[5] + Linv[3] + Uinv[7] + v; }
}
}}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
  for (int w = 0; w < 3; ++w) hdg::bench_diag<<<1, 32>>>(out, cyc, 50, w);
  long long h[8];
  cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
  printf("diag_factor %lld cycles, diag_inverses %lld, inv_times_tile %lld\n", h[0], h[1], h[2]);
  return 0;
}
