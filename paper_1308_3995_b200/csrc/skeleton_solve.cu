// skeleton_solve.cu — SURVEY.md §8(f) NEXT #3: the skeleton solve that consumes K and E ("First, the hybridized
// system is assembled and then being solved for dLambda"; "In our code we use an ILU(n)-
// preconditioned GMRES which is available through the PETSc library").
//
// B200 form: restarted GMRES(m), right-preconditioned (the Arnoldi residual estimate is the true residual), with a
// block-Jacobi preconditioner — the inverses of K's diagonal blocks (one dense n_fp x n_fp block per face row, a
// warp-level Gauss-Jordan with partial pivoting each) — instead of ILU(n), whose triangular sweeps serialise on a
// GPU. Every vector operation is one of the kernels below; the host holds only the (m+1) x m Hessenberg matrix and
// its Givens rotations. Classical Gram-Schmidt with one re-orthogonalisation pass, deterministic reductions (fixed
// block partition, fixed-order second pass: no floating-point atomics), so a solve is bitwise reproducible.
#include <algorithm>
#include <cmath>
#include <vector>

#include "dev_common.cuh"
#include "hdg_internal.cuh"

namespace hdg {
namespace {

constexpr int kRedBlocks = 296;   // 2 x 148 SMs: the fixed partition of every reduction
constexpr int kRedThreads = 256;

// y[rows of owned face f] = sum over the blocks of row f of K_block * x[cols]. RPW block rows per warp (RPW = 2 when
// every face has <= 16 trace dofs: half-warps, no idle lanes on C4's 16-dof faces); lane r of a (half-)warp owns
// row r of its block row.
template <int RPW>
__global__ void __launch_bounds__(256) spmv_kernel(const double* K, const double* x, double* y, const int32_t* row_ptr,
                                                   const int32_t* col_idx, const int64_t* blk_off,
                                                   const int32_t* face_ndof, const int64_t* face_off, int64_t f0,
                                                   int64_t nrows, int64_t tr0) {
  constexpr int W = 32 / RPW;
  const int lane = threadIdx.x & (W - 1);
  const int64_t r = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * RPW + ((threadIdx.x & 31) / W);
  if (r >= nrows) return;
  const int64_t f = f0 + r;
  const int nr = face_ndof[f];
  double acc = 0.0;
  for (int q = row_ptr[r]; q < row_ptr[r + 1]; ++q) {
    const int c = col_idx[q];
    const int nc = face_ndof[c];
    const double* Kb = K + blk_off[q];
    const double* xc = x + face_off[c];
    if (lane < nr)
      for (int j = 0; j < nc; ++j) acc = fma(__ldg(Kb + lane * nc + j), __ldg(xc + j), acc);
  }
  if (lane < nr) y[face_off[f] - tr0 + lane] = acc;
}

// Dinv_f = K_ff^-1 for every owned face (Gauss-Jordan with partial pivoting on [K_ff | I] in the warp's shared
// memory slice; lanes stride over the 2 n columns; n <= kMaxFaceSolve). A singular diagonal block leaves an identity block (the
// preconditioner then skips that row; GMRES still converges on the unpreconditioned row).
__global__ void __launch_bounds__(128) bjacobi_setup_kernel(const double* K, double* Dinv, const int32_t* row_ptr,
                                                            const int32_t* col_idx, const int64_t* blk_off,
                                                            const int32_t* face_ndof, const int64_t* dinv_off,
                                                            int64_t f0, int64_t nrows) {
  __shared__ double M_s[4][kMaxFaceSolve * 49];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * 4 + w;
  if (r >= nrows) return;
  const int64_t f = f0 + r;
  const int n = face_ndof[f];
  double* M = M_s[w];
  constexpr int ld = 49;   // [K_ff | I]: 2 n <= 48 columns
  int q = row_ptr[r];
  const int qe = row_ptr[r + 1];
  while (q < qe && col_idx[q] != (int32_t)f) ++q;   // the diagonal block (present in every owned row)
  if (q == qe) {   // (defensive: no diagonal block — the preconditioner skips the row)
    double* D = Dinv + dinv_off[r];
    for (int i = 0; i < n; ++i)
      for (int j = lane; j < n; j += 32) D[i * n + j] = i == j ? 1.0 : 0.0;
    return;
  }
  const double* Kb = K + blk_off[q];
  for (int i = 0; i < n; ++i) {
    for (int j = lane; j < 2 * n; j += 32) M[i * ld + j] = j < n ? Kb[i * n + j] : (j - n == i ? 1.0 : 0.0);
  }
  __syncwarp();
  bool sing = false;
  for (int k = 0; k < n; ++k) {
    double best = lane >= k && lane < n ? fabs(M[lane * ld + k]) : -1.0;
    int bi = lane;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (!(best > 0.0)) { sing = true; break; }
    if (bi != k)
      for (int j = lane; j < 2 * n; j += 32) {
        const double t = M[k * ld + j];
        M[k * ld + j] = M[bi * ld + j];
        M[bi * ld + j] = t;
      }
    __syncwarp();
    const double rp = 1.0 / M[k * ld + k];
    for (int j = lane; j < 2 * n; j += 32) M[k * ld + j] *= rp;
    __syncwarp();
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const double l = M[i * ld + k];
      for (int j = lane; j < 2 * n; j += 32) M[i * ld + j] = fma(-l, M[k * ld + j], M[i * ld + j]);
    }
    __syncwarp();
  }
  double* D = Dinv + dinv_off[r];
  for (int i = 0; i < n; ++i)
    for (int j = lane; j < n; j += 32) D[i * n + j] = sing ? (i == j ? 1.0 : 0.0) : M[i * ld + n + j];
}

// out[rows of f] = Dinv_f in[rows of f] (owned rows; local trace numbering)
__global__ void __launch_bounds__(256) bjacobi_apply_kernel(const double* Dinv, const double* in, double* out,
                                                            const int32_t* face_ndof, const int64_t* face_off,
                                                            const int64_t* dinv_off, int64_t f0, int64_t nrows,
                                                            int64_t tr0) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= nrows) return;
  const int64_t f = f0 + r;
  const int n = face_ndof[f];
  const int64_t o = face_off[f] - tr0;
  if (lane < n) {
    const double* D = Dinv + dinv_off[r] + lane * n;
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc = fma(D[j], in[o + j], acc);
    out[o + lane] = acc;
  }
}

// partial[j][b] = sum over block b's fixed index range of V_j . w, j < k (V: k vectors of length n, stride ldv)
__global__ void __launch_bounds__(kRedThreads) dots_partial_kernel(const double* V, int64_t ldv, int k, const double* w,
                                                                   int64_t n, double* partial) {
  __shared__ double red[kRedThreads / 32][32];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  for (int j0 = 0; j0 < k; j0 += 32) {
    const int jn = min(32, k - j0);
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const double wi = w[i];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < jn) acc[j] = fma(V[(int64_t)(j0 + j) * ldv + i], wi, acc[j]);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      double v = acc[j];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) red[wp][j] = v;
    }
    __syncthreads();
    if (threadIdx.x < jn) {
      double s = 0.0;
      for (int q = 0; q < kRedThreads / 32; ++q) s += red[q][threadIdx.x];
      partial[(int64_t)(j0 + threadIdx.x) * gridDim.x + blockIdx.x] = s;
    }
    __syncthreads();
  }
}

// h[j] = sum over blocks (fixed order) of partial[j][b]
__global__ void dots_final_kernel(const double* partial, int k, int nblocks, double* h) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += partial[(int64_t)j * nblocks + b];
  h[j] = s;
}

// w -= sum_j h[j] V_j   (or out = sum_j h[j] V_j when accumulate == false)
__global__ void __launch_bounds__(256) combine_kernel(const double* V, int64_t ldv, int k, const double* h, double* w,
                                                      int64_t n, bool subtract) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int j = 0; j < k; ++j) acc = fma(h[j], V[(int64_t)j * ldv + i], acc);
  w[i] = subtract ? w[i] - acc : acc;
}

// y = alpha x + beta y
__global__ void __launch_bounds__(256) axpby_kernel(double alpha, const double* x, double beta, double* y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = alpha * x[i] + beta * y[i];
}

// halo exchange of the distributed solve: gather the sent trace dofs, scatter the received ones
__global__ void __launch_bounds__(256) gather_kernel(const double* x, const int64_t* idx, int64_t n, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = x[idx[i]];
}
__global__ void __launch_bounds__(256) scatter_kernel(const double* in, const int64_t* idx, int64_t n, double* x) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[idx[i]] = in[i];
}

unsigned nb(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace

// The solver (host loop over the kernels above). Single rank: x (global trace vector) is the whole unknown.
cudaError_t skeleton_gmres(const Plan& p, SolverWork& sw, const double* K, const double* E, double* x, double rtol,
                           int maxit, int m, cudaStream_t s, int* iters, double* relres, int64_t* launches,
                           void* comm, int rank, int nranks, std::string* comm_err) {
  const Skeleton& k = p.sk;
  const int64_t n = k.ntr, nrows = k.f1 - k.f0;
  const bool dist = comm != nullptr && nranks > 1;
  cudaError_t e;
  // ---- workspace (kept in the plan across solves)
  if (sw.n != n || sw.m != m) {
    cudaFree(sw.V); cudaFree(sw.w); cudaFree(sw.z); cudaFree(sw.partial); cudaFree(sw.h); cudaFree(sw.Dinv);
    cudaFree(sw.dinv_off);
    cudaFree(sw.xfull); cudaFree(sw.hsend); cudaFree(sw.hrecv); cudaFree(sw.d_hsend_idx); cudaFree(sw.d_hrecv_idx);
    sw = SolverWork();
    std::vector<int64_t> doff(nrows + 1, 0);
    std::vector<int32_t> fnd(p.F);
    if ((e = cudaMemcpy(fnd.data(), p.d_face_ndof, sizeof(int32_t) * p.F, cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
    for (int64_t r = 0; r < nrows; ++r) doff[r + 1] = doff[r] + (int64_t)fnd[k.f0 + r] * fnd[k.f0 + r];
    if ((e = cudaMalloc(&sw.V, sizeof(double) * (size_t)(m + 1) * std::max<int64_t>(n, 1))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&sw.w, sizeof(double) * std::max<int64_t>(n, 1))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&sw.z, sizeof(double) * std::max<int64_t>(n, 1))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&sw.partial, sizeof(double) * (size_t)(m + 2) * kRedBlocks)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&sw.h, sizeof(double) * (size_t)(m + 2))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&sw.Dinv, sizeof(double) * std::max<int64_t>(doff[nrows], 1))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&sw.dinv_off, sizeof(int64_t) * (nrows + 1))) != cudaSuccess) return e;
    if ((e = cudaMemcpy(sw.dinv_off, doff.data(), sizeof(int64_t) * (nrows + 1), cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    sw.n = n;
    sw.m = m;
  }
  if (dist && !sw.halo_built) {
    sw.n_hsend = (int64_t)p.halo_send_idx.size();
    sw.n_hrecv = (int64_t)p.halo_recv_idx.size();
    if ((e = cudaMalloc(&sw.xfull, sizeof(double) * std::max<int64_t>(p.n_trace, 1))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&sw.hsend, sizeof(double) * std::max<int64_t>(sw.n_hsend, 1))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&sw.hrecv, sizeof(double) * std::max<int64_t>(sw.n_hrecv, 1))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&sw.d_hsend_idx, sizeof(int64_t) * std::max<int64_t>(sw.n_hsend, 1))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&sw.d_hrecv_idx, sizeof(int64_t) * std::max<int64_t>(sw.n_hrecv, 1))) != cudaSuccess) return e;
    if (sw.n_hsend && (e = cudaMemcpy(sw.d_hsend_idx, p.halo_send_idx.data(), sizeof(int64_t) * sw.n_hsend,
                                      cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    if (sw.n_hrecv && (e = cudaMemcpy(sw.d_hrecv_idx, p.halo_recv_idx.data(), sizeof(int64_t) * sw.n_hrecv,
                                      cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    sw.halo_built = true;
  }
  *iters = 0;
  *relres = 0.0;
  // (a rank without owned rows still takes part in every collective below)
  if (n == 0 && !dist) return cudaSuccess;
  bool comm_ok = true;
  // the halo of a full-length vector: my owned dofs that others' rows read, then theirs into mine
  auto halo = [&](double* xf) {
    if (!dist || !comm_ok) return;
    if (sw.n_hsend) gather_kernel<<<nb(sw.n_hsend, 256), 256, 0, s>>>(xf, sw.d_hsend_idx, sw.n_hsend, sw.hsend);
    comm_ok = nccl_p2p(comm, rank, nranks, p.halo_scnt, p.halo_sdsp, sw.hsend, p.halo_rcnt, p.halo_rdsp, sw.hrecv, s,
                       comm_err);
    if (sw.n_hrecv) scatter_kernel<<<nb(sw.n_hrecv, 256), 256, 0, s>>>(sw.hrecv, sw.d_hrecv_idx, sw.n_hrecv, xf);
    *launches += 2;
  };
  const int64_t ldv = n;
  double* V = sw.V;
  const int32_t* rp = k.d_row_ptr;
  auto spmv = [&](const double* xin, double* y) {
    if (nrows == 0) return;
    if (p.max_face_ndof <= 16)
      spmv_kernel<2><<<nb(nrows, 16), 256, 0, s>>>(K, xin, y, rp, k.d_col_idx, k.d_blk_off, p.d_face_ndof,
                                                   p.d_face_off, k.f0, nrows, k.tr0);
    else
      spmv_kernel<1><<<nb(nrows, 8), 256, 0, s>>>(K, xin, y, rp, k.d_col_idx, k.d_blk_off, p.d_face_ndof,
                                                   p.d_face_off, k.f0, nrows, k.tr0);
    ++*launches;
  };
  // K v for an owned-length vector v: v into the full-length work vector, its halo, then the SpMV
  auto spmv_v = [&](const double* v, double* y) {
    if (!dist) {
      spmv(v, y);
      return;
    }
    if (n) cudaMemcpyAsync(sw.xfull + k.tr0, v, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
    halo(sw.xfull);
    spmv(sw.xfull, y);
  };
  auto prec = [&](const double* in, double* out) {
    if (nrows == 0) return;
    bjacobi_apply_kernel<<<nb(nrows, 8), 256, 0, s>>>(sw.Dinv, in, out, p.d_face_ndof, p.d_face_off, sw.dinv_off,
                                                      k.f0, nrows, k.tr0);
    ++*launches;
  };
  // h[0..kk) = V[0..kk)^T w  (device h, then host copy)
  std::vector<double> hh(m + 2);
  auto dots = [&](const double* Vb, int kk, const double* w, double* host) -> cudaError_t {
    dots_partial_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(Vb, ldv, kk, w, n, sw.partial);
    dots_final_kernel<<<nb(kk, 64), 64, 0, s>>>(sw.partial, kk, kRedBlocks, sw.h);
    *launches += 2;
    if (dist && comm_ok) comm_ok = nccl_allreduce_sum(comm, sw.h, (size_t)kk, s, comm_err);   // sum over slabs
    if (!comm_ok) return cudaErrorUnknown;
    cudaError_t er = cudaMemcpyAsync(host, sw.h, sizeof(double) * kk, cudaMemcpyDeviceToHost, s);
    if (er == cudaSuccess) er = cudaStreamSynchronize(s);
    return er;
  };
  if (nrows > 0) {
    bjacobi_setup_kernel<<<nb(nrows, 4), 128, 0, s>>>(K, sw.Dinv, rp, k.d_col_idx, k.d_blk_off, p.d_face_ndof,
                                                      sw.dinv_off, k.f0, nrows);
    ++*launches;
  }
  double* xo = x + k.tr0;   // this rank's owned part of lambda (the whole vector on one rank)
  // ||E||
  double bn = 0.0;
  if ((e = dots(E, 1, E, &bn)) != cudaSuccess) return e;
  bn = std::sqrt(bn);
  if (bn == 0.0) {
    cudaMemsetAsync(x, 0, sizeof(double) * p.n_trace, s);
    return cudaStreamSynchronize(s);
  }
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
  int total = 0;
  double res = 0.0;
  while (total < maxit) {
    // r = E - K x  -> V_0 (x: the caller's full-length lambda; its halo refreshed first)
    halo(x);
    spmv(x, sw.w);
    axpby_kernel<<<nb(n, 256), 256, 0, s>>>(1.0, E, -1.0, sw.w, n);
    ++*launches;
    double beta = 0.0;
    if ((e = dots(sw.w, 1, sw.w, &beta)) != cudaSuccess) return e;
    beta = std::sqrt(beta);
    res = beta / bn;
    if (res <= rtol) break;
    axpby_kernel<<<nb(n, 256), 256, 0, s>>>(1.0 / beta, sw.w, 0.0, V, n);
    ++*launches;
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int j = 0;
    for (; j < m && total < maxit; ++j, ++total) {
      prec(V + (int64_t)j * ldv, sw.z);
      spmv_v(sw.z, sw.w);
      // classical Gram-Schmidt, twice (re-orthogonalisation)
      if ((e = dots(V, j + 1, sw.w, hh.data())) != cudaSuccess) return e;
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = hh[i];
      combine_kernel<<<nb(n, 256), 256, 0, s>>>(V, ldv, j + 1, sw.h, sw.w, n, true);
      ++*launches;
      if ((e = dots(V, j + 1, sw.w, hh.data())) != cudaSuccess) return e;
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] += hh[i];
      combine_kernel<<<nb(n, 256), 256, 0, s>>>(V, ldv, j + 1, sw.h, sw.w, n, true);
      ++*launches;
      double hn = 0.0;
      if ((e = dots(sw.w, 1, sw.w, &hn)) != cudaSuccess) return e;
      hn = std::sqrt(hn);
      H[(size_t)(j + 1) * m + j] = hn;
      if (hn > 0.0) {
        axpby_kernel<<<nb(n, 256), 256, 0, s>>>(1.0 / hn, sw.w, 0.0, V + (int64_t)(j + 1) * ldv, n);
        ++*launches;
      }
      // Givens rotations on column j
      for (int i = 0; i < j; ++i) {
        const double a = H[(size_t)i * m + j], b = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * a + sn[i] * b;
        H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * b;
      }
      const double a = H[(size_t)j * m + j], b = H[(size_t)(j + 1) * m + j];
      const double rr = std::hypot(a, b);
      cs[j] = rr > 0.0 ? a / rr : 1.0;
      sn[j] = rr > 0.0 ? b / rr : 0.0;
      H[(size_t)j * m + j] = rr;
      H[(size_t)(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      res = std::fabs(g[j + 1]) / bn;
      if (res <= rtol || hn == 0.0) { ++j; ++total; break; }
    }
    // x += M^-1 V y, H y = g (upper triangular j x j)
    for (int i = j - 1; i >= 0; --i) {
      double t = g[i];
      for (int c = i + 1; c < j; ++c) t -= H[(size_t)i * m + c] * y[c];
      y[i] = t / H[(size_t)i * m + i];
    }
    if ((e = cudaMemcpyAsync(sw.h, y.data(), sizeof(double) * j, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
    combine_kernel<<<nb(n, 256), 256, 0, s>>>(V, ldv, j, sw.h, sw.w, n, false);
    prec(sw.w, sw.z);
    axpby_kernel<<<nb(n, 256), 256, 0, s>>>(1.0, sw.z, 1.0, xo, n);
    *launches += 2;
    if (res <= rtol) break;
  }
  // every rank's owned segment to all ranks (lambda replicated, as the back-substitution reads it), then the true
  // residual of the returned x
  if (dist && comm_ok) comm_ok = nccl_allgatherv_inplace(comm, nranks, p.rank_tr0, p.rank_ntr, x, s, comm_err);
  if (!comm_ok) return cudaErrorUnknown;
  spmv(x, sw.w);
  axpby_kernel<<<nb(n, 256), 256, 0, s>>>(1.0, E, -1.0, sw.w, n);
  ++*launches;
  double rt = 0.0;
  if ((e = dots(sw.w, 1, sw.w, &rt)) != cudaSuccess) return e;
  *relres = std::sqrt(rt) / bn;
  *iters = total;
  return cudaGetLastError();
}

cudaError_t skeleton_spmv(const Plan& p, const double* K, const double* x, double* y, cudaStream_t s,
                          int64_t* launches) {
  const Skeleton& k = p.sk;
  const int64_t nrows = k.f1 - k.f0;
  if (nrows <= 0) return cudaSuccess;
  if (p.max_face_ndof <= 16)
    spmv_kernel<2><<<nb(nrows, 16), 256, 0, s>>>(K, x, y, k.d_row_ptr, k.d_col_idx, k.d_blk_off, p.d_face_ndof,
                                                 p.d_face_off, k.f0, nrows, k.tr0);
  else
    spmv_kernel<1><<<nb(nrows, 8), 256, 0, s>>>(K, x, y, k.d_row_ptr, k.d_col_idx, k.d_blk_off, p.d_face_ndof,
                                                 p.d_face_off, k.f0, nrows, k.tr0);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace hdg
