#include <cstdio>
__device__ __forceinline__ double fast_rcp(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;\n" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
template <int MODE>
__device__ __noinline__ bool fwd(double* Dg, int ldT, double* buf, int lane, long long* st) {
  const int j = lane & 15; const bool dl = lane < 16;
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = dl ? Dg[i * ldT + j] : ((i == j) ? 1.0 : 0.0);
  bool viol = false;
  double rnext = fast_rcp(x[0]);
  long long t0 = clock64();
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    double* bc = buf + (c & 1) * 16;
    if (MODE != 1) {
    if (lane == c) {
      const double pv = x[c];
#pragma unroll
      for (int i = c + 1; i < 16; ++i) { viol |= fabs(x[i]) > fabs(pv); const double m = x[i] * rnext; x[i] = m; bc[i] = m; }
    }
    __syncwarp();
    }
    const double xc = x[c];
    if (!dl || j > c) {
      if (c + 1 < 16) { x[c + 1] = fma(-bc[c + 1], xc, x[c + 1]); if (MODE != 2) rnext = fast_rcp(x[c + 1]); }
#pragma unroll
      for (int i = c + 2; i < 16; ++i) x[i] = fma(-bc[i], xc, x[i]);
    }
  }
  long long t1 = clock64();
  if (lane == 0) st[MODE] = t1 - t0;
#pragma unroll
  for (int i = 0; i < 16; ++i) Dg[i * ldT + j] = x[i];
  return viol;
}
__global__ void k(double* out, long long* st) {
  __shared__ double T[16 * 20], buf[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < 320; i += 32) T[i] = (i % 21 == 0) ? 4.0 : 0.01 * (i % 7);
  __syncwarp();
  bool v = fwd<0>(T, 20, buf, lane, st); __syncwarp();
  for (int i = lane; i < 320; i += 32) T[i] = (i % 21 == 0) ? 4.0 : 0.01 * (i % 7);
  v |= fwd<1>(T, 20, buf, lane, st); __syncwarp();
  for (int i = lane; i < 320; i += 32) T[i] = (i % 21 == 0) ? 4.0 : 0.01 * (i % 7);
  v |= fwd<2>(T, 20, buf, lane, st);
  out[lane] = T[lane] + v;
}
int main() {
  double* out; long long* st; cudaMalloc(&out, 512); cudaMalloc(&st, 64);
  k<<<1, 32>>>(out, st); k<<<1, 32>>>(out, st);
  long long h[4]; cudaMemcpy(h, st, 32, cudaMemcpyDeviceToHost);
  printf("forward full %lld | no lane-c region %lld | no rcp %lld\n", h[0], h[1], h[2]);
}
