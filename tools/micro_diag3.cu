// 2D-layout (8 row-pairs x 4 column-octets of [D | I]) diagonal-block factorization with shared-memory broadcast.
#include <cstdio>
#include <cmath>
__device__ __forceinline__ double fast_rcp(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;\n" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
constexpr int NB = 16, LDI = 20;
// bc: broadcast buffer >= 2 x 48 doubles
template <int MODE>
__device__ __noinline__ bool diag2d(double* Dg, int ldT, double* Linv, double* Uinv, double* bc, int lane) {
  const int rg = lane >> 2, cg = lane & 3;
  const bool isD = cg < 2;
  const int col0 = 8 * (cg & 1);         // first D or I column of this lane
  double v[2][8];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int r = 2 * rg + q;
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      double2 t = isD ? *reinterpret_cast<const double2*>(Dg + r * ldT + col0 + k) : make_double2(0.0, 0.0);
      if (!isD) { t.x = (r == col0 + k) ? 1.0 : 0.0; t.y = (r == col0 + k + 1) ? 1.0 : 0.0; }
      v[q][k] = t.x; v[q][k + 1] = t.y;
    }
  }
  bool viol = false;
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    double* b = bc + (c & 1) * 48;        // [0,32): pivot row c (32 cols of [D|I]); [32,48): column c of D
    // publish: lanes of row group c>>1 write row c (their 8 columns); lanes of column octet c>>3 write column c
    if (!(MODE & 2)) {
    if (rg == (c >> 1)) {
#pragma unroll
      for (int k = 0; k < 8; k += 2) *reinterpret_cast<double2*>(b + 8 * cg + k) = make_double2(v[c & 1][k], v[c & 1][k + 1]);
    }
    if (cg == (c >> 3)) *reinterpret_cast<double2*>(b + 32 + 2 * rg) = make_double2(v[0][c & 7], v[1][c & 7]);
    __syncwarp();
    }
    const double pv = b[8 * (c >> 3) + (c & 7)];
    const double rp = fast_rcp(pv);
    const double2 ac = *reinterpret_cast<const double2*>(b + 32 + 2 * rg);
    double prow[8];
#pragma unroll
    for (int k = 0; k < 8; k += 2) { const double2 t = *reinterpret_cast<const double2*>(b + 8 * cg + k); prow[k] = t.x; prow[k + 1] = t.y; }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = 2 * rg + q;
      const double a = q ? ac.y : ac.x;
      const bool below = r > c;
      viol |= below && (fabs(a) > fabs(pv));
      const double l = below ? a * rp : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int col = col0 + k;
        const bool keep = isD && col <= c;          // L part / pivot column of D: no row operation
        const double nv = fma(-l, prow[k], v[q][k]);
        v[q][k] = keep ? ((col == c && below) ? l : v[q][k]) : nv;
      }
    }
  }
  viol |= false;
  // L\U -> Dg, L^-1 -> Linv
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int r = 2 * rg + q;
    double* dst = isD ? Dg + r * ldT + col0 : Linv + r * LDI + col0;
#pragma unroll
    for (int k = 0; k < 8; k += 2) *reinterpret_cast<double2*>(dst + k) = make_double2(v[q][k], v[q][k + 1]);
  }
  if (MODE & 1) return __any_sync(0xffffffffu, viol);
  // backward Gauss-Jordan on [U | I] -> U^-1 (identity half restarted; D half keeps U)
  double rd[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int r = 2 * rg + q;
    rd[q] = fast_rcp(Dg[r * ldT + r]);   // written above by the owner lane; same warp, ordered by syncwarp below
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int r = 2 * rg + q;
    rd[q] = fast_rcp(Dg[r * ldT + r]);
#pragma unroll
    for (int k = 0; k < 8; ++k) if (!isD) v[q][k] = (r == col0 + k) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int c = NB - 1; c >= 0; --c) {
    double* b = bc + (c & 1) * 48;
    if (rg == (c >> 1) && !isD) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[c & 1][k] *= rd[c & 1];
#pragma unroll
      for (int k = 0; k < 8; k += 2) *reinterpret_cast<double2*>(b + 8 * cg + k) = make_double2(v[c & 1][k], v[c & 1][k + 1]);
    }
    if (cg == (c >> 3)) *reinterpret_cast<double2*>(b + 32 + 2 * rg) = make_double2(v[0][c & 7], v[1][c & 7]);
    __syncwarp();
    if (!isD) {
      const double2 uc = *reinterpret_cast<const double2*>(b + 32 + 2 * rg);
      double prow[8];
#pragma unroll
      for (int k = 0; k < 8; k += 2) { const double2 t = *reinterpret_cast<const double2*>(b + 8 * cg + k); prow[k] = t.x; prow[k + 1] = t.y; }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = 2 * rg + q;
        const double u = (r < c) ? (q ? uc.y : uc.x) : 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) v[q][k] = fma(-u, prow[k], v[q][k]);
      }
    }
  }
  if (!isD) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = 2 * rg + q;
#pragma unroll
      for (int k = 0; k < 8; k += 2) *reinterpret_cast<double2*>(Uinv + r * LDI + col0 + k) = make_double2(v[q][k], v[q][k + 1]);
    }
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
  for (int m = 3; m >= 0; --m) {
  long long acc = 0;
  for (int r = 0; r < 20; ++r) {
    for (int i = lane; i < 320; i += 32) T[i] = T0[i];
    __syncwarp();
    long long t0 = clock64();
    if (m == 0) v |= diag2d<0>(T, 20, Li, Ui, bc, lane);
    if (m == 1) v |= diag2d<1>(T, 20, Li, Ui, bc, lane);
    if (m == 2) v |= diag2d<2>(T, 20, Li, Ui, bc, lane);
    if (m == 3) v |= diag2d<3>(T, 20, Li, Ui, bc, lane);
    __syncwarp();
    { long long dt = clock64() - t0; if (rr_min_ok(dt)) {} acc = (acc == 0 || dt < acc) ? dt : acc; }
  }
  st[m] = acc;
  }
  // verification: L U == D (as in T0), Li * L == I, Ui * U == I
  if (lane == 0) {
    double e1 = 0, e2 = 0, e3 = 0;
    for (int i = 0; i < 16; ++i) for (int j = 0; j < 16; ++j) {
      double s = 0; for (int k = 0; k < 16; ++k) { double L = (i == k) ? 1.0 : (k < i ? T[i * 20 + k] : 0.0); double U = (k <= j) ? T[k * 20 + j] : 0.0; s += L * U; }
      e1 = fmax(e1, fabs(s - T0[i * 20 + j]));
      double s2 = 0; for (int k = 0; k < 16; ++k) { double L = (k == j) ? 1.0 : (j < k ? T[k * 20 + j] : 0.0); s2 += Li[i * 20 + k] * L; }
      e2 = fmax(e2, fabs(s2 - (i == j)));
      double s3 = 0; for (int k = 0; k < 16; ++k) { double U = (k <= j) ? T[k * 20 + j] : 0.0; s3 += Ui[i * 20 + k] * U; }
      e3 = fmax(e3, fabs(s3 - (i == j)));
    }
    out[0] = e1; out[1] = e2; out[2] = e3; out[3] = v;
  }
}
int main() {
  double* out; long long* st; cudaMalloc(&out, 512); cudaMalloc(&st, 64);
  k<<<1, 32>>>(out, st); cudaDeviceSynchronize();
  long long hh[4]; double e[4]; cudaMemcpy(hh, st, 32, cudaMemcpyDeviceToHost); cudaMemcpy(e, out, 32, cudaMemcpyDeviceToHost);
  long long h = hh[0];
  printf("full %lld fwd-only %lld no-publish %lld fwd-no-publish %lld\n", hh[0], hh[1], hh[2], hh[3]);
  printf("diag2d %lld cycles | |LU-D| %.2e |Linv L - I| %.2e |Uinv U - I| %.2e viol %g\n", h, e[0], e[1], e[2], e[3]);
}
