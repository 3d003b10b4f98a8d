// Cycles of the chain warp's per-panel work outside diag_chain: prep_next (L21/U12 tiles of the next diagonal
// block, 8 DMMA chains) and the 16x16 update of that block (upd_block), one warp alone on the SM.
#include "../../paper_1308_3995_b200/csrc/condense_sweep.cu"
#include <cstdio>
namespace hdg { namespace {
__global__ void bench(double* LUg, long long* cyc) {
  extern __shared__ double sm[];
  const int ld = 180;
  double* T = sm;                    // 64 x 180
  double* Li = T + 64 * ld;
  double* Ui = Li + 16 * LDI;
  const int lane = threadIdx.x;
  for (int i = lane; i < 64 * ld; i += 32) T[i] = 0.01 * ((i * 7) % 13) - 0.06;
  for (int i = lane; i < 16 * LDI; i += 32) { Li[i] = (i % LDI == i / LDI) ? 1.0 : 0.01; Ui[i] = Li[i]; }
  __syncwarp();
  long long b1 = 1LL << 60, b2 = 1LL << 60, b3 = 1LL << 60;
  for (int r = 0; r < 10; ++r) {
    long long t0 = clock64();
    bool v = prep_next(T, ld, 0, 16, 16, 32, 16, Li, Ui, LUg, 120, lane);
    long long t1 = clock64();
    upd_block(T, ld, T, ld, T, ld, 16, 2, 16, 2, 16, lane);
    __syncwarp();
    long long t2 = clock64();
    upd_block(T, ld, T, ld, T, ld, 32, 2, 32, 4, 16, lane);
    __syncwarp();
    long long t3 = clock64();
    b1 = min(b1, t1 - t0); b2 = min(b2, t2 - t1); b3 = min(b3, t3 - t2);
    if (v) cyc[7] = 1;
  }
  if (lane == 0) { cyc[0] = b1; cyc[1] = b2; cyc[2] = b3; }
}
}}
int main() {
  double* LUg; long long* cyc; cudaMalloc(&LUg, 120 * 120 * 8); cudaMalloc(&cyc, 64);
  cudaFuncSetAttribute(hdg::bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
  hdg::bench<<<1, 32, 120000>>>(LUg, cyc); cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
  printf("prep_next %lld cycles | upd 16x16 k16 %lld | upd 16x32 k16 %lld  (%s)\n", h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
}
