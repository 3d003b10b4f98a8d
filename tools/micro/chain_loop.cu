// The chain warp's per-panel loop (prep_next -> 16x16 update -> diag_chain) of condense_sweep.cu run by one warp
// on a C4-sized working matrix: per-phase cycles in a loop, to compare with the same functions timed alone.
#include "../../paper_1308_3995_b200/csrc/condense_sweep.cu"
#include <cstdio>
namespace hdg { namespace {
__global__ void bench(double* LUg, long long* cyc, int nwarps_busy) {
  extern __shared__ double sm[];
  const int ld = 180, ne = 120;
  double* T = sm;
  double* Li = T + 120 * ld;
  double* Ui = Li + 2 * 16 * LDI;
  double* bc = Ui + 2 * 16 * LDI;
  const int lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
  for (int i = threadIdx.x; i < 120 * ld; i += blockDim.x) {
    const int r = i / ld, c = i % ld;
    T[i] = (r == c) ? 3.0 : 0.3 * sin(0.1 * i) / 11.0;
  }
  __syncthreads();
  if (warp == blockDim.x / 32 - 1) {
    long long tp = 0, tu = 0, td = 0;
    bool v = diag_chain(T, ld, 0, 16, Li, Ui, bc, LUg, ne, lane);
    for (int p = 0; p < 7; ++p) {
      const int jb = 16 * p, jn = jb + 16, nn = min(16, ne - jn), nn8 = (nn + 7) & ~7;
      long long t0 = clock64();
      v |= prep_next(T, ld, jb, 16, jn, min(jn + 16, 120), nn8, Li + (p & 1) * 16 * LDI, Ui + (p & 1) * 16 * LDI, LUg, ne, lane);
      long long t1 = clock64();
      upd_block(T, ld, T + jb, ld, T + (size_t)jb * ld, ld, jn, nn8 >> 3, jn, nn8 >> 3, 16, lane);
      __syncwarp();
      long long t2 = clock64();
      v |= diag_chain(T, ld, jn, nn, Li + ((p + 1) & 1) * 16 * LDI, Ui + ((p + 1) & 1) * 16 * LDI, bc, LUg, ne, lane);
      long long t3 = clock64();
      tp += t1 - t0; tu += t2 - t1; td += t3 - t2;
    }
    if (lane == 0) { cyc[0] = tp / 7; cyc[1] = tu / 7; cyc[2] = td / 7; cyc[3] = v; }
  }
}
}}
int main() {
  double* LUg; long long* cyc; cudaMalloc(&LUg, 120 * 120 * 8); cudaMalloc(&cyc, 64);
  cudaFuncSetAttribute(hdg::bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  for (int smem : {232448, 225000, 215000, 200000, 190000}) {
    // the carveout: the shared-memory size sets how much of the unified L1 is left
    hdg::bench<<<1, 32, smem>>>(LUg, cyc, 1); cudaDeviceSynchronize();
    long long h[4]; cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    printf("smem %6d B: prep %lld | update %lld | diag %lld  (viol %lld, %s)\n", smem, h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
  }
}
