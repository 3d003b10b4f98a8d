// Rows layout: lane r < 16 holds D row r, lane 16 + r holds row r of the identity part. Pivot rows are final
// when published, so they are written straight to their outputs (T for U, Linv for L^-1) and read back as
// broadcasts. U^-1: lanes = columns, right-looking backward substitution with broadcast loads of U.
#include <cstdio>
#include <cmath>
__device__ __forceinline__ double fast_rcp(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;\n" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
constexpr int NB = 16, LDI = 20;
__device__ __noinline__ bool diag_rows(double* Dg, int ldT, double* Linv, double* Uinv, double* rcpbuf, int lane) {
  const int r = lane & 15;
  const bool isD = lane < 16;
  double x[NB];
  double* myrow = isD ? Dg + r * ldT : Linv + r * LDI;
#pragma unroll
  for (int j = 0; j < NB; j += 2) {
    double2 t = isD ? *reinterpret_cast<const double2*>(myrow + j) : make_double2(j == r ? 1.0 : 0.0, j + 1 == r ? 1.0 : 0.0);
    x[j] = t.x; x[j + 1] = t.y;
  }
  bool viol = false;
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    // owner lanes (D row c, I row c) publish their final rows
    if (r == c) {
#pragma unroll
      for (int j = 0; j < NB; j += 2)
        if (isD ? (j + 1 >= c) : (j <= c)) *reinterpret_cast<double2*>(myrow + j) = make_double2(x[j], x[j + 1]);
    }
    __syncwarp();
    const double* prow = isD ? Dg + c * ldT : Linv + c * LDI;
    const double pv = Dg[c * ldT + c];
    double l = 0.0;
    if (isD) {
      viol |= (r > c) && (fabs(x[c]) > fabs(pv));
      l = x[c] * fast_rcp(pv);
    }
    l = __shfl_sync(0xffffffffu, l, r);
    if (r > c) {
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if (isD ? (j > c) : (j <= c)) x[j] = fma(-l, prow[j], x[j]);
      }
      if (isD) x[c] = l;
    }
  }
  // rows r > ... : write remaining (non-pivot) parts: D rows hold L in j < r (multipliers) ; all rows were
  // published when they were pivots except the L parts of D rows, written here
  if (isD) {
#pragma unroll
    for (int j = 0; j < NB; j += 2)
      if (j < r) *reinterpret_cast<double2*>(myrow + j) = make_double2(x[j], (j + 1 < r) ? x[j + 1] : myrow[j + 1]);
  }
  // 1/u_jj for the backward substitution
  if (isD) rcpbuf[r] = fast_rcp(x[r]);
  __syncwarp();
  // U^-1 by columns: lane j < 16 solves U y = e_j, right-looking from the bottom
  if (isD) {
    const int j = r;
    double y[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) y[i] = (i == j) ? 1.0 : 0.0;
#pragma unroll
    for (int k = NB - 1; k >= 0; --k) {
      y[k] *= rcpbuf[k];
#pragma unroll
      for (int i = 0; i < k; ++i) y[i] = fma(-Dg[i * ldT + k], y[k], y[i]);
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) Uinv[i * LDI + j] = y[i];
  }
  return __any_sync(0xffffffffu, viol);
}
__device__ __forceinline__ bool rr_min_ok(long long) { return true; }
__global__ void k(double* out, long long* st) {
  __shared__ __align__(16) double T[16 * 20], T0[16 * 20], Li[16 * 20], Ui[16 * 20], bc[96];
  const int lane = threadIdx.x;
  for (int i = lane; i < 320; i += 32) T0[i] = ((i % 20) == (i / 20)) ? 4.0 + 0.1 * (i / 20) : 0.01 * ((i * 7) % 11) - 0.05;
  __syncwarp();
  bool v = false;
  long long acc = 0;
  for (int rr = 0; rr < 20; ++rr) {
    for (int i = lane; i < 320; i += 32) T[i] = T0[i];
    __syncwarp();
    long long t0 = clock64();
    v |= diag_rows(T, 20, Li, Ui, bc, lane);
    __syncwarp();
    { long long dt = clock64() - t0; if (rr_min_ok(dt)) {} acc = (acc == 0 || dt < acc) ? dt : acc; }
  }
  st[0] = acc;
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
    out[0] = e1; out[1] = e2; out[2] = e3; out[3] = v;
  }
}
int main() {
  double* out; long long* st; cudaMalloc(&out, 512); cudaMalloc(&st, 64);
  k<<<1, 32>>>(out, st); cudaDeviceSynchronize();
  long long h; double e[4]; cudaMemcpy(&h, st, 8, cudaMemcpyDeviceToHost); cudaMemcpy(e, out, 32, cudaMemcpyDeviceToHost);
  printf("diag_rows %lld cycles | |LU-D| %.2e |Linv L - I| %.2e |Uinv U - I| %.2e viol %g\n", h, e[0], e[1], e[2], e[3]);
}
