// Variants of the 16x16 diagonal-block chain (LU + L^-1 + U^-1 in one loop), one warp, clock64 — to pick the
// fastest formulation for condense_sweep.cu. Each variant checks its own factors.
#include <cstdio>
#include <cmath>
constexpr int NB = 16, LDI = 20, BCW = 36;
__device__ __forceinline__ double rcp_fast(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;\n" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0); const double t = fma(e, e, e); return fma(r, t, r);
}
// MODE bits: 1 = include L^-1 (e) part, 2 = shuffles instead of smem broadcast, 4 = lane c publishes row
// progressively right after each FMA (smem mode)
template <int MODE>
__device__ __forceinline__ void chain(double* T, int ld, double* Linv, double* Uinv, double* bc, int lane) {
  const bool lo = lane < 16;
  const int r = lane & 15;
  double d[NB], e[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) { d[j] = lo ? T[r * ld + j] : 0.0; e[j] = (lo && j == r) ? 1.0 : 0.0; }
  if (!(MODE & 2)) {
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < NB; ++j) bc[j] = d[j];
      bc[16] = e[0];
    }
  }
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    double u[NB], pe[NB];
    if (MODE & 2) {
#pragma unroll
      for (int j = c; j < NB; ++j) u[j] = __shfl_sync(0xffffffffu, d[j], c);
      if (MODE & 1) {
#pragma unroll
        for (int j = 0; j <= c; ++j) pe[j] = __shfl_sync(0xffffffffu, e[j], c);
      }
    } else {
      const double* slot = bc + (c & 1) * BCW;
      __syncwarp();
#pragma unroll
      for (int j = c; j < NB; ++j) u[j] = slot[j];
      if (MODE & 1) {
#pragma unroll
        for (int j = 0; j <= c; ++j) pe[j] = slot[16 + j];
      }
    }
    const double rp = rcp_fast(u[c]);
    const bool lrow = lo && r > c, urow = !lo && r <= c;
    const double dc = d[c];
    const double l = dc * rp;
    const double zr = (r == c ? 1.0 : -dc) * rp;
    const double coef = lrow ? -l : (urow ? zr : 0.0);
    double* nslot = bc + ((c + 1) & 1) * BCW;
    const bool me = lane == c + 1;
#pragma unroll
    for (int j = c + 1; j < NB; ++j) {
      d[j] = fma(coef, u[j], d[j]);
      if ((MODE & 4) && !(MODE & 2) && me) nslot[j] = d[j];
    }
    if (MODE & 1) {
      const double ce = lrow ? -l : 0.0;
#pragma unroll
      for (int j = 0; j <= c; ++j) e[j] = fma(ce, pe[j], e[j]);
    }
    if (lrow) d[c] = l;
    if (urow) e[c] = zr;
    if (!(MODE & 2) && c + 1 < NB && me) {
      if (!(MODE & 4)) {
#pragma unroll
        for (int j = c + 1; j < NB; ++j) nslot[j] = d[j];
      }
#pragma unroll
      for (int j = 0; j <= c + 1; ++j) nslot[16 + j] = e[j];
    }
  }
  if (lo) {
#pragma unroll
    for (int j = 0; j < NB; ++j) { T[r * ld + j] = d[j]; Linv[r * LDI + j] = e[j]; }
  } else {
#pragma unroll
    for (int j = 0; j < NB; ++j) Uinv[r * LDI + j] = e[j];
  }
  __syncwarp();
}
template <int MODE>
__global__ void bench(double* out, long long* cyc) {
  __shared__ __align__(16) double T[16 * 20], T0[16 * 20], Li[16 * 20], Ui[16 * 20], bc[2 * BCW];
  const int lane = threadIdx.x;
  for (int i = lane; i < 320; i += 32) T0[i] = ((i % 20) == (i / 20)) ? 4.0 + 0.1 * (i / 20) : 0.01 * ((i * 7) % 11) - 0.05;
  __syncwarp();
  long long best = 1LL << 60, first = 0;
  for (int rr = 0; rr < 20; ++rr) {
    for (int i = lane; i < 320; i += 32) T[i] = T0[i];
    __syncwarp();
    long long t0 = clock64();
    chain<MODE>(T, 20, Li, Ui, bc, lane);
    long long dt = clock64() - t0;
    best = dt < best ? dt : best;
    if (rr == 0) first = dt;
  }
  if (lane == 0) {
    double e1 = 0, e2 = 0, e3 = 0;
    for (int i = 0; i < 16; ++i) for (int j = 0; j < 16; ++j) {
      double s = 0; for (int kk = 0; kk < 16; ++kk) { double L = (i == kk) ? 1.0 : (kk < i ? T[i * 20 + kk] : 0.0); double U = (kk <= j) ? T[kk * 20 + j] : 0.0; s += L * U; }
      e1 = fmax(e1, fabs(s - T0[i * 20 + j]));
      double s2 = 0; for (int kk = 0; kk < 16; ++kk) { double L = (kk == j) ? 1.0 : (j < kk ? T[kk * 20 + j] : 0.0); s2 += Li[i * 20 + kk] * L; }
      e2 = fmax(e2, fabs(s2 - (i == j)));
      double s3 = 0; for (int kk = 0; kk < 16; ++kk) { double U = (kk <= j) ? T[kk * 20 + j] : 0.0; s3 += Ui[i * 20 + kk] * U; }
      e3 = fmax(e3, fabs(s3 - (i == j)));
    }
    printf("MODE %d: first (cold I-cache) %lld, best %lld cycles | |LU-A| %.1e |Linv L-I| %.1e |Uinv U-I| %.1e\n", MODE, first, best, e1, (MODE & 1) ? e2 : 0.0, e3);
  }
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
  bench<0><<<1, 32>>>(out, cyc); cudaDeviceSynchronize();
  bench<1><<<1, 32>>>(out, cyc); cudaDeviceSynchronize();
  bench<2><<<1, 32>>>(out, cyc); cudaDeviceSynchronize();
  bench<3><<<1, 32>>>(out, cyc); cudaDeviceSynchronize();
  bench<4><<<1, 32>>>(out, cyc); cudaDeviceSynchronize();
  bench<5><<<1, 32>>>(out, cyc); cudaDeviceSynchronize();
  return 0;
}
