// Which hardware warp slot (%warpid; SMSP = slot mod 4) does each warp of two co-resident CTAs get?
#include <cstdio>
#include <vector>
__global__ void k(int* out) {
  extern __shared__ double sm[];
  unsigned s, w;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(w));
  if ((threadIdx.x & 31) == 0) {
    int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    out[3 * i] = s; out[3 * i + 1] = w; out[3 * i + 2] = blockIdx.x;
  }
  sm[threadIdx.x] = s;
  for (volatile int i = 0; i < 100000; ++i) {}
}
int main() {
  const int nb = 296, nt = 256, smem = 100 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int* d; cudaMalloc(&d, nb * 8 * 3 * 4);
  k<<<nb, nt, smem>>>(d);
  cudaDeviceSynchronize();
  std::vector<int> h(nb * 8 * 3);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  for (int sm = 0; sm < 3; ++sm) {
    printf("SM %d:", sm);
    for (int i = 0; i < nb * 8; ++i) if (h[3 * i] == sm) printf(" b%d.w%d->%d", h[3 * i + 2], i % 8, h[3 * i + 1]);
    printf("\n");
  }
  int odd = 0, tot = 0;
  for (int b = 0; b < nb; ++b) { int w0 = h[3 * (b * 8) + 1]; odd += (w0 >> 3) & 1; ++tot; }
  printf("CTAs whose warp 0 is in an odd group of 8 slots: %d / %d\n", odd, tot);
}
