// lu8 (condense_sweep.cu) vs a 2-D-distributed variant: lane (q, r) holds a[r][2q..2q+1] of the 8x8 block (4
// shuffles per elimination step instead of 9), the triangular inverses afterwards by column-parallel substitution
// from shared memory (lanes 0-7: L^-1 columns, lanes 8-15: U^-1 columns through the row/column reversal).
#include "../../paper_1308_3995_b200/csrc/condense_sweep.cu"
#include <cstdio>
namespace hdg { namespace {
__device__ __forceinline__ bool lu8v2(double* X, int ld, int r0, int nbv, double* Li8, double* Ui8, double* LU, int ne,
                                      int lane, long long* tk) {
  long long ta = clock64();
  __syncwarp();
  const int r = lane & 7, q = lane >> 3;
  double x0, x1;
  {
    const bool real = r < nbv;
    double2 v = make_double2(0.0, 0.0);
    if (real && 2 * q < nbv) v = *reinterpret_cast<const double2*>(X + (size_t)(r0 + r) * ld + r0 + 2 * q);
    x0 = real ? (2 * q < nbv ? v.x : 0.0) : (2 * q == r ? 1.0 : 0.0);
    x1 = real ? (2 * q + 1 < nbv ? v.y : 0.0) : (2 * q + 1 == r ? 1.0 : 0.0);
  }
  bool viol = false;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double v = (c & 1) ? x1 : x0;
    const int cq = c >> 1;
    const double piv = __shfl_sync(0xffffffffu, v, 8 * cq + c);
    const double arc = __shfl_sync(0xffffffffu, v, 8 * cq + r);
    const double u0 = __shfl_sync(0xffffffffu, x0, 8 * q + c);
    const double u1 = __shfl_sync(0xffffffffu, x1, 8 * q + c);
    const double rp = rcp_fast(piv);
    const double l = arc * rp;
    const bool lrow = r > c;
    viol |= lrow && fabs(arc) > fabs(piv);
    viol |= r == c && pivot_bad(piv);
    const int j0 = 2 * q, j1 = 2 * q + 1;
    if (lrow) {
      x0 = j0 > c ? fma(-l, u0, x0) : (j0 == c ? l : x0);
      x1 = j1 > c ? fma(-l, u1, x1) : (j1 == c ? l : x1);
    }
  }
  long long tb = clock64();
  if (r < nbv && 2 * q < nbv) {
    *reinterpret_cast<double2*>(X + (size_t)(r0 + r) * ld + r0 + 2 * q) = make_double2(x0, x1);
    *reinterpret_cast<double2*>(LU + (size_t)(r0 + r) * ne + r0 + 2 * q) = make_double2(x0, x1);
  }
  // padded rows / columns of the block are identity: keep them in a private copy for the substitutions
  __shared__ double Mb[8 * 8];
  Mb[r * 8 + 2 * q] = x0;
  Mb[r * 8 + 2 * q + 1] = x1;
  __syncwarp();
  long long tc = clock64();
  // forward substitution for column j of M^-1, M lower triangular: lanes 0-7 M = L (unit), lanes 8-15
  // M = J U J (J = reversal), lanes 16-31 duplicate 0-15 (results discarded)
  const bool isU = (lane & 8) != 0;
  const int j = lane & 7;
  double y[8], dinv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    y[k] = k == j ? 1.0 : 0.0;
    const double rk = rcp_fast(Mb[(7 - k) * 9]);
    dinv[k] = isU ? rk : 1.0;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    y[k] *= dinv[k];
#pragma unroll
    for (int i = k + 1; i < 8; ++i) {
      const double m = Mb[isU ? (7 - i) * 8 + 7 - k : i * 8 + k];
      y[i] = fma(-m, y[k], y[i]);
    }
  }
  if (lane < 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) Li8[i * LDI + j] = y[i];
  } else if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 8; ++i) Ui8[(7 - i) * LDI + 7 - j] = y[i];
  }
  __syncwarp();
  long long td = clock64();
  if (lane == 0) { tk[0] = tb - ta; tk[1] = tc - tb; tk[2] = td - tc; }
  return __any_sync(0xffffffffu, viol);
}

__device__ __forceinline__ bool lu8v3(double* X, int ld, int r0, int nbv, double* Li8, double* Ui8, double* LU, int ne,
                                      int lane, long long* tk) {
  long long ta = clock64();
  __syncwarp();
  const int r = lane & 7, q = lane >> 3;
  double x0, x1;
  {
    const bool real = r < nbv;
    double2 v = make_double2(0.0, 0.0);
    if (real && 2 * q < nbv) v = *reinterpret_cast<const double2*>(X + (size_t)(r0 + r) * ld + r0 + 2 * q);
    x0 = real ? (2 * q < nbv ? v.x : 0.0) : (2 * q == r ? 1.0 : 0.0);
    x1 = real ? (2 * q + 1 < nbv ? v.y : 0.0) : (2 * q + 1 == r ? 1.0 : 0.0);
  }
  bool viol = false;
#pragma unroll
  for (int c = 0; c < 8; c += 2) {
    // steps c and c+1 fused: pivot block [[p00 p01] [p10 p11]] = rows c, c+1 x columns c, c+1 (lane (c/2, c), (c/2, c+1))
    const int cq = c >> 1;
    const double p00 = __shfl_sync(0xffffffffu, x0, 8 * cq + c);
    const double p01 = __shfl_sync(0xffffffffu, x1, 8 * cq + c);
    const double p10 = __shfl_sync(0xffffffffu, x0, 8 * cq + c + 1);
    const double p11 = __shfl_sync(0xffffffffu, x1, 8 * cq + c + 1);
    const double ar0 = __shfl_sync(0xffffffffu, x0, 8 * cq + r);   // a[r][c]
    const double ar1 = __shfl_sync(0xffffffffu, x1, 8 * cq + r);   // a[r][c+1]
    const double uc0 = __shfl_sync(0xffffffffu, x0, 8 * q + c);     // row c at this lane's columns
    const double uc1 = __shfl_sync(0xffffffffu, x1, 8 * q + c);
    const double ud0 = __shfl_sync(0xffffffffu, x0, 8 * q + c + 1); // row c+1 at this lane's columns
    const double ud1 = __shfl_sync(0xffffffffu, x1, 8 * q + c + 1);
    const double rp0 = rcp_fast(p00);
    const double l10 = p10 * rp0;                 // multiplier of row c+1 at step c
    const double lr0 = ar0 * rp0;                 // multiplier of row r at step c
    const double up11 = fma(-l10, p01, p11);      // pivot of step c+1
    const double ar1p = fma(-lr0, p01, ar1);      // a[r][c+1] after step c
    const double rp1 = rcp_fast(up11);
    const double lr1 = ar1p * rp1;                // multiplier of row r at step c+1
    const double ue0 = fma(-l10, uc0, ud0);       // row c+1 after step c, this lane's columns
    const double ue1 = fma(-l10, uc1, ud1);
    viol |= (r > c) && fabs(ar0) > fabs(p00);
    viol |= (r > c + 1) && fabs(ar1p) > fabs(up11);
    viol |= r == c && pivot_bad(p00);
    viol |= r == c + 1 && pivot_bad(up11);
    const int j0 = 2 * q, j1 = 2 * q + 1;
    if (r == c + 1) {
      x0 = j0 > c ? ue0 : (j0 == c ? l10 : x0);
      x1 = j1 > c ? ue1 : (j1 == c ? l10 : x1);
    } else if (r > c + 1) {
      x0 = j0 > c + 1 ? fma(-lr1, ue0, fma(-lr0, uc0, x0)) : (j0 == c ? lr0 : (j0 == c + 1 ? lr1 : x0));
      x1 = j1 > c + 1 ? fma(-lr1, ue1, fma(-lr0, uc1, x1)) : (j1 == c ? lr0 : (j1 == c + 1 ? lr1 : x1));
    }
  }
  long long tb = clock64();
  if (r < nbv && 2 * q < nbv) {
    *reinterpret_cast<double2*>(X + (size_t)(r0 + r) * ld + r0 + 2 * q) = make_double2(x0, x1);
    *reinterpret_cast<double2*>(LU + (size_t)(r0 + r) * ne + r0 + 2 * q) = make_double2(x0, x1);
  }
  // padded rows / columns of the block are identity: keep them in a private copy for the substitutions
  __shared__ double Mb[8 * 8];
  Mb[r * 8 + 2 * q] = x0;
  Mb[r * 8 + 2 * q + 1] = x1;
  __syncwarp();
  long long tc = clock64();
  // forward substitution for column j of M^-1, M lower triangular: lanes 0-7 M = L (unit), lanes 8-15
  // M = J U J (J = reversal), lanes 16-31 duplicate 0-15 (results discarded)
  const bool isU = (lane & 8) != 0;
  const int j = lane & 7;
  double y[8], dinv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    y[k] = k == j ? 1.0 : 0.0;
    const double rk = rcp_fast(Mb[(7 - k) * 9]);
    dinv[k] = isU ? rk : 1.0;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    y[k] *= dinv[k];
#pragma unroll
    for (int i = k + 1; i < 8; ++i) {
      const double m = Mb[isU ? (7 - i) * 8 + 7 - k : i * 8 + k];
      y[i] = fma(-m, y[k], y[i]);
    }
  }
  if (lane < 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) Li8[i * LDI + j] = y[i];
  } else if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 8; ++i) Ui8[(7 - i) * LDI + 7 - j] = y[i];
  }
  __syncwarp();
  long long td = clock64();
  if (lane == 0) { tk[0] = tb - ta; tk[1] = tc - tb; tk[2] = td - tc; }
  return __any_sync(0xffffffffu, viol);
}


// v4: lane = 4r + q (the m8n8 accumulator layout), branch-free selects, L^-1 / U^-1 by column substitution
__device__ __forceinline__ bool lu8v4(double* X, int ld, int r0, int nbv, double* Li8, double* Ui8, double* LU, int ne,
                                      int lane, long long* tk) {
  long long ta = clock64();
  __syncwarp();
  const int r = lane >> 2, q = lane & 3;
  const int j0 = 2 * q, j1 = 2 * q + 1;
  double x0, x1;
  {
    const bool real = r < nbv;
    double2 v = make_double2(0.0, 0.0);
    if (real && j0 < nbv) v = *reinterpret_cast<const double2*>(X + (size_t)(r0 + r) * ld + r0 + j0);
    x0 = real ? (j0 < nbv ? v.x : 0.0) : (j0 == r ? 1.0 : 0.0);
    x1 = real ? (j1 < nbv ? v.y : 0.0) : (j1 == r ? 1.0 : 0.0);
  }
  bool viol = false;
  double rps[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double v = (c & 1) ? x1 : x0;
    const double piv = __shfl_sync(0xffffffffu, v, 4 * c + (c >> 1));
    const double arc = __shfl_sync(0xffffffffu, v, 4 * r + (c >> 1));
    const double u0 = __shfl_sync(0xffffffffu, x0, 4 * c + q);
    const double u1 = __shfl_sync(0xffffffffu, x1, 4 * c + q);
    const double rp = rcp_fast(piv);
    rps[c] = rp;
    const double l = arc * rp;
    const bool lrow = r > c;
    viol |= lrow & (fabs(arc) > fabs(piv));
    viol |= (r == c) & pivot_bad(piv);
    const double n0 = fma(-l, u0, x0), n1 = fma(-l, u1, x1);
    const bool g0 = lrow & (j0 > c), e0 = lrow & (j0 == c);
    const bool g1 = lrow & (j1 > c), e1 = lrow & (j1 == c);
    x0 = g0 ? n0 : x0;
    x0 = e0 ? l : x0;
    x1 = g1 ? n1 : x1;
    x1 = e1 ? l : x1;
  }
  long long tb = clock64();
  if (r < nbv && j0 < nbv) {
    *reinterpret_cast<double2*>(X + (size_t)(r0 + r) * ld + r0 + j0) = make_double2(x0, x1);
    *reinterpret_cast<double2*>(LU + (size_t)(r0 + r) * ne + r0 + j0) = make_double2(x0, x1);
  }
  __shared__ __align__(16) double Mb4[8 * 8];
  *reinterpret_cast<double2*>(Mb4 + r * 8 + j0) = make_double2(x0, x1);
  __syncwarp();
  long long tc = clock64();
  const bool isU = (lane & 8) != 0;
  const int j = lane & 7;
  double m[8][8], y[8], dinv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    dinv[k] = isU ? rps[7 - k] : 1.0;
    y[k] = k == j ? 1.0 : 0.0;
#pragma unroll
    for (int i = k + 1; i < 8; ++i) m[i][k] = Mb4[isU ? (7 - i) * 8 + 7 - k : i * 8 + k];
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    y[k] *= dinv[k];
#pragma unroll
    for (int i = k + 1; i < 8; ++i) y[i] = fma(-m[i][k], y[k], y[i]);
  }
  double* dst = isU ? Ui8 + 7 - j : Li8 + j;
  const int rs = isU ? -LDI : LDI;
  double* d0 = isU ? dst + 7 * LDI : dst;
  if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 8; ++i) d0[i * rs] = y[i];
  }
  __syncwarp();
  long long td = clock64();
  if (lane == 0) { tk[0] = tb - ta; tk[1] = tc - tb; tk[2] = td - tc; }
  return __any_sync(0xffffffffu, viol);
}

__global__ void bench(double* LUg, long long* cyc, double* out, int mode) {
  __shared__ __align__(16) double T[16 * 20], T0[16 * 20], Li[16 * LDI], Ui[16 * LDI], St[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < 320; i += 32) T0[i] = ((i % 20) == (i / 20)) ? 4.0 + 0.1 * (i / 20) : 0.31 * sin(1.7 * i);
  for (int i = lane; i < 16 * LDI; i += 32) { Li[i] = 0.0; Ui[i] = 0.0; }
  __syncwarp();
  long long best = 1LL << 60;
  bool v = false;
  for (int rep = 0; rep < 20; ++rep) {
    for (int i = lane; i < 320; i += 32) T[i] = T0[i];
    __syncwarp();
    long long t0 = clock64();
    if (mode == 0) v |= lu8(T, 20, 0, 8, Li, Ui, LUg, 16, St, lane);
    else if (mode == 1) v |= lu8v2(T, 20, 0, 8, Li, Ui, LUg, 16, lane, cyc + 4);
    else if (mode == 2) v |= lu8v3(T, 20, 0, 8, Li, Ui, LUg, 16, lane, cyc + 4);
    else v |= lu8v4(T, 20, 0, 8, Li, Ui, LUg, 16, lane, cyc + 4);
    long long dt = clock64() - t0;
    best = dt < best ? dt : best;
  }
  for (int i = lane; i < 64; i += 32) {
    out[i] = T[(i / 8) * 20 + i % 8];
    out[64 + i] = Li[(i / 8) * LDI + i % 8];
    out[128 + i] = Ui[(i / 8) * LDI + i % 8];
  }
  if (lane == 0) { cyc[0] = best; cyc[1] = v; }
}
}}
int main() {
  double *LUg, *out; long long* cyc;
  cudaMalloc(&LUg, 256 * 8); cudaMalloc(&cyc, 64); cudaMalloc(&out, 4 * 192 * 8);
  double h[4][192];
  for (int m = 0; m < 4; ++m) {
    hdg::bench<<<1, 32>>>(LUg, cyc, out + 192 * m, m); cudaDeviceSynchronize();
    long long c[8]; cudaMemcpy(c, cyc, 64, cudaMemcpyDeviceToHost);
    if (m) printf("  lu loop %lld | store+stage %lld | inverses %lld\n", c[4], c[5], c[6]);
    cudaMemcpy(h[m], out + 192 * m, 192 * 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %lld cycles, viol %lld, %s\n", m, m == 3 ? "lu8v4" : m == 2 ? "lu8v3" : m ? "lu8v2" : "lu8", c[0], c[1], cudaGetErrorString(cudaGetLastError()));
  }
  for (int m = 1; m < 4; ++m) {
    double md = 0; for (int i = 0; i < 192; ++i) md = fmax(md, fabs(h[0][i] - h[m][i]));
    printf("max |lu8 - mode %d| over LU, L^-1, U^-1: %.3e\n", m, md);
  }
}
