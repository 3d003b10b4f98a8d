// Phase breakdown of diag_chain (condense_sweep.cu) run by one warp: lu8 #1 | L21/U12 | D22 update | lu8 #2 |
// inverse assembly, in cycles, averaged over 7 diagonal blocks of a C4-sized working matrix.
#include "../../paper_1308_3995_b200/csrc/condense_sweep.cu"
#include <cstdio>
namespace hdg { namespace {
__global__ void bench(double* LUg, long long* cyc) {
  extern __shared__ double sm[];
  const int ldT = 180, ne = 120;
  double* T = sm;
  double* Lb = T + 120 * ldT;
  double* Ub = Lb + 2 * 16 * LDI;
  double* St = Ub + 2 * 16 * LDI;
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 120 * ldT; i += blockDim.x) {
    const int r = i / ldT, c = i % ldT;
    T[i] = (r == c) ? 3.0 : 0.3 * sin(0.1 * i) / 11.0;
  }
  __syncthreads();
  long long t[6] = {0, 0, 0, 0, 0, 0};
  bool viol = false;
  for (int p = 0; p < 7; ++p) {
    const int jb = 16 * p;
    double* Linv = Lb + (p & 1) * 16 * LDI;
    double* Uinv = Ub + (p & 1) * 16 * LDI;
    double* LU = LUg;
    __syncwarp();
    long long c0 = clock64();
    viol |= lu8(T, ldT, jb, 8, Linv, Uinv, LU, ne, St, lane);
    long long c1 = clock64();
    const int gid = lane >> 2, tig = lane & 3, c = 2 * tig;
    double* D12 = T + (size_t)jb * ldT + jb + 8;
    double* D21 = T + (size_t)(jb + 8) * ldT + jb;
    double* D22 = D21 + 8;
    double l21[2] = {0.0, 0.0}, u12[2] = {0.0, 0.0};
    mm8(l21, D21, ldT, Uinv, LDI, 1.0, lane);
    mm8(u12, Linv, LDI, D12, ldT, 1.0, lane);
    __syncwarp();
    viol |= fabs(l21[0]) > 1.0 || fabs(l21[1]) > 1.0;
    st8(D21, ldT, l21, lane);
    *reinterpret_cast<double2*>(LU + (size_t)(jb + 8 + gid) * ne + jb + c) = make_double2(l21[0], l21[1]);
    *reinterpret_cast<double2*>(D12 + gid * ldT + c) = make_double2(u12[0], u12[1]);
    *reinterpret_cast<double2*>(LU + (size_t)(jb + gid) * ne + jb + 8 + c) = make_double2(u12[0], u12[1]);
    __syncwarp();
    long long c2 = clock64();
    double d22[2];
    d22[0] = D22[gid * ldT + c];
    d22[1] = D22[gid * ldT + c + 1];
    mm8(d22, D21, ldT, D12, ldT, -1.0, lane);
    __syncwarp();
    *reinterpret_cast<double2*>(D22 + gid * ldT + c) = make_double2(d22[0], d22[1]);
    __syncwarp();
    long long c3 = clock64();
    viol |= lu8(T, ldT, jb + 8, 8, Linv + 8 * LDI + 8, Uinv + 8 * LDI + 8, LU, ne, St, lane);
    long long c4 = clock64();
    double P[2] = {0.0, 0.0}, Q[2] = {0.0, 0.0};
    mm8(P, D21, ldT, Linv, LDI, 1.0, lane);
    mm8(Q, D12, ldT, Uinv + 8 * LDI + 8, LDI, 1.0, lane);
    st8(Linv + 8 * LDI, LDI, P, lane);
    st8(Uinv + 8, LDI, Q, lane);
    *reinterpret_cast<double2*>(Linv + gid * LDI + 8 + c) = make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(Uinv + (8 + gid) * LDI + c) = make_double2(0.0, 0.0);
    __syncwarp();
    double X[2] = {0.0, 0.0}, Y[2] = {0.0, 0.0};
    mm8(X, Linv + 8 * LDI + 8, LDI, Linv + 8 * LDI, LDI, -1.0, lane);
    mm8(Y, Uinv, LDI, Uinv + 8, LDI, -1.0, lane);
    __syncwarp();
    st8(Linv + 8 * LDI, LDI, X, lane);
    st8(Uinv + 8, LDI, Y, lane);
    __syncwarp();
    viol = __any_sync(0xffffffffu, viol);
    long long c5 = clock64();
    t[0] += c1 - c0; t[1] += c2 - c1; t[2] += c3 - c2; t[3] += c4 - c3; t[4] += c5 - c4; t[5] += c5 - c0;
  }
  if (lane == 0) for (int i = 0; i < 6; ++i) cyc[i] = t[i] / 7;
  if (lane == 0) cyc[6] = viol;
}
}}
int main() {
  double* LUg; long long* cyc; cudaMalloc(&LUg, 120 * 120 * 8); cudaMalloc(&cyc, 64);
  cudaFuncSetAttribute(hdg::bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  for (int rep = 0; rep < 2; ++rep) {
    hdg::bench<<<1, 32, 200000>>>(LUg, cyc); cudaDeviceSynchronize();
    long long h[7]; cudaMemcpy(h, cyc, 56, cudaMemcpyDeviceToHost);
    printf("lu8 %lld | L21/U12 %lld | D22 %lld | lu8 %lld | inverses %lld | total %lld (viol %lld, %s)\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6], cudaGetErrorString(cudaGetLastError()));
  }
}
