// skeleton.cu — rows a0 (symbolic part), a6 and a7 of the hot path: the skeleton system.
//
// "The hybridized matrix is an n_f x n_f block matrix ... In each block row there is one block on the diagonal
//  and 2d off-diagonal blocks in the case of simplex elements. These blocks represent the edges of the
//  neighboring elements of one edge.". K and E collect the element contributions S_e, g_e
// (Eq. hybridsystem), assembled element-wise.
//
// a0 symbolic (once per plan): per owned face row, the sorted union of the faces of its left and right
//    elements -> row_ptr (block counts), col_idx (ascending), blk_off (int64 running sum of block sizes).
//    Integer-only, bit-exact; the two prefix sums are a hand-written single-CTA scan.
// a6 numeric: gather form — every K block is written by exactly one warp, which reads the <= 2 contributing
//    S_e sub-blocks (left element first, then right) and sums them in that fixed order; no atomics, so the
//    result is deterministic and bitwise equal to the oracle's left-then-right sum.
// a7 exchange pack / accumulate for faces shared between element slabs (nranks > 1).
#include "hdg_internal.cuh"

namespace hdg {
namespace {

__device__ __forceinline__ int row_cols(const int32_t* elem_face, const int32_t* face_elem, int64_t f, int32_t (&cols)[6]) {
  int nc = 0;
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const int32_t e = face_elem[2 * f + side];
    if (e < 0) continue;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int32_t c = elem_face[3 * (int64_t)e + k];
      if (c < 0) continue;
      bool dup = false;
      for (int q = 0; q < nc; ++q) dup |= cols[q] == c;
      if (!dup) cols[nc++] = c;
    }
  }
  for (int a = 1; a < nc; ++a)
    for (int b = a; b > 0 && cols[b - 1] > cols[b]; --b) { const int32_t t = cols[b]; cols[b] = cols[b - 1]; cols[b - 1] = t; }
  return nc;
}

__global__ void sym_count_kernel(const int32_t* elem_face, const int32_t* face_elem, const int32_t* face_ndof, int64_t f0,
                                 int64_t nrows, int64_t* cnt, int64_t* vals) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int32_t cols[6];
  const int nc = row_cols(elem_face, face_elem, f0 + r, cols);
  int64_t v = 0;
  for (int q = 0; q < nc; ++q) v += (int64_t)face_ndof[f0 + r] * face_ndof[cols[q]];
  cnt[r] = nc;
  vals[r] = v;
}

// exclusive scan of n int64 values into out[0..n] (out[n] = total); one CTA of 1024 threads
__global__ void __launch_bounds__(1024) scan_kernel(const int64_t* in, int64_t n, int64_t* out) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t chunk = (n + 1023) / 1024;
  const int64_t b = t * chunk, e = min(n, b + chunk);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += in[i];
  part[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int64_t v = t >= off ? part[t - off] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = part[t] - s;   // exclusive prefix of this thread's chunk
  for (int64_t i = b; i < e; ++i) { out[i] = run; run += in[i]; }
  if (t == 1023) out[n] = part[1023];
}

__global__ void sym_fill_kernel(const int32_t* elem_face, const int32_t* face_elem, const int32_t* face_ndof, int64_t f0,
                                int64_t nrows, const int64_t* row_start, const int64_t* val_start, int32_t* row_ptr,
                                int32_t* col_idx, int64_t* blk_off, int32_t* blk_row) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r > nrows) return;
  row_ptr[r] = (int32_t)row_start[r];
  if (r == nrows) { blk_off[row_start[r]] = val_start[r]; return; }
  int32_t cols[6];
  const int nc = row_cols(elem_face, face_elem, f0 + r, cols);
  int64_t q = row_start[r], v = val_start[r];
  for (int c = 0; c < nc; ++c, ++q) {
    col_idx[q] = cols[c];
    blk_row[q] = (int32_t)(f0 + r);
    blk_off[q] = v;
    v += (int64_t)face_ndof[f0 + r] * face_ndof[cols[c]];
  }
}

struct AsmArgs {
  const double *S, *g;
  double *K, *E;
  const int32_t *elem_face, *face_elem, *face_ndof, *nf;
  const int64_t *face_off, *offS, *offG;
  const int32_t *col_idx, *blk_row;
  const int64_t* blk_off;
  int64_t eb, n, nnzb, f0, f1, tr0;
};

// slot of face f in element e (global ids) and the offset of that slot in e's trace ordering
__device__ __forceinline__ int slot_of(const int32_t* elem_face, const int32_t* face_ndof, int64_t e, int32_t f, int* soff) {
  int o = 0, s = -1;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int32_t c = elem_face[3 * e + k];
    if (c == f && s < 0) { s = k; *soff = o; }
    if (c >= 0) o += face_ndof[c];
  }
  return s;
}

// a6: one warp per K block; left contribution first, then right: K = (0 + S_left) + S_right.
// TR (adjoint): K~ = sum_e S_e^T, i.e. block (f, f') takes S_e[slot f' rows, slot f cols]^T.
template <bool TR>
__global__ void __launch_bounds__(256) assemble_kernel(const AsmArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (q >= a.nnzb) return;
  const int32_t f = a.blk_row[q], c = a.col_idx[q];
  const int na = a.face_ndof[f], nb = a.face_ndof[c];
  // the (at most two) contributing elements, left first; scalars, not arrays indexed by the running count (those
  // went to local memory)
  const double *src0 = nullptr, *src1 = nullptr;
  int ld0 = 0, ld1 = 0, ns = 0;
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const int32_t e = a.face_elem[2 * (int64_t)f + side];
    if (e < a.eb || e >= a.eb + a.n) continue;   // -1 or not local
    int so_a = 0, so_b = 0;
    if (slot_of(a.elem_face, a.face_ndof, e, f, &so_a) < 0) continue;
    if (slot_of(a.elem_face, a.face_ndof, e, c, &so_b) < 0) continue;
    const int64_t l = e - a.eb;
    const int ldl = a.nf[l];
    const double* sp = TR ? a.S + a.offS[l] + (int64_t)so_b * ldl + so_a : a.S + a.offS[l] + (int64_t)so_a * ldl + so_b;
    if (ns == 0) { src0 = sp; ld0 = ldl; } else { src1 = sp; ld1 = ldl; }
    ++ns;
  }
  double* dst = a.K + a.blk_off[q];
  int r = lane / nb, cc = lane - (lane / nb) * nb;   // (r, cc) of idx, advanced by 32 without divisions
  const int step_r = 32 / nb, step_c = 32 - (32 / nb) * nb;
  for (int idx = lane; idx < na * nb; idx += 32) {
    double v = 0.0;
    if (ns > 0) v = v + __ldg(TR ? src0 + (int64_t)cc * ld0 + r : src0 + (int64_t)r * ld0 + cc);
    if (ns > 1) v = v + __ldg(TR ? src1 + (int64_t)cc * ld1 + r : src1 + (int64_t)r * ld1 + cc);
    dst[idx] = v;
    r += step_r;
    cc += step_c;
    if (cc >= nb) {
      cc -= nb;
      ++r;
    }
  }
}

// a6 right-hand side: E[f] = (0 + g_left) + g_right, one warp per owned face
__global__ void __launch_bounds__(256) assemble_rhs_kernel(const AsmArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t f = a.f0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (f >= a.f1) return;
  const int na = a.face_ndof[f];
  const double *src0 = nullptr, *src1 = nullptr;
  int ns = 0;
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const int32_t e = a.face_elem[2 * f + side];
    if (e < a.eb || e >= a.eb + a.n) continue;
    int so = 0;
    if (slot_of(a.elem_face, a.face_ndof, e, (int32_t)f, &so) < 0) continue;
    const double* sp = a.g + a.offG[e - a.eb] + so;
    if (ns == 0) src0 = sp; else src1 = sp;
    ++ns;
  }
  double* dst = a.E + (a.face_off[f] - a.tr0);
  for (int i = lane; i < na; i += 32) {
    double v = 0.0;
    if (ns > 0) v = v + __ldg(src0 + i);
    if (ns > 1) v = v + __ldg(src1 + i);
    dst[i] = v;
  }
}

// a7 pack: item (face f, local element l, offset o): send[o .. o+na) = g_l[slot f], then the na x nf_l strip
// S_l[slot f rows, all columns] (row-major). One warp per item. TR (adjoint): the strip of S_l^T, i.e. S_l's
// slot-f columns, so that the owner's ordered accumulate builds K~ = sum S_e^T exactly as K.
template <bool TR>
__global__ void __launch_bounds__(256) pack_kernel(const AsmArgs a, const int64_t* items, int64_t n_items, double* send) {
  const int lane = threadIdx.x & 31;
  const int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (it >= n_items) return;
  const int32_t f = (int32_t)items[3 * it];
  const int64_t l = items[3 * it + 1], o = items[3 * it + 2];
  const int64_t e = a.eb + l;
  int so = 0;
  slot_of(a.elem_face, a.face_ndof, e, f, &so);
  const int na = a.face_ndof[f], nfl = a.nf[l];
  const double* g = a.g + a.offG[l] + so;
  const double* S = a.S + a.offS[l] + (TR ? so : (int64_t)so * nfl);
  for (int i = lane; i < na; i += 32) send[o + i] = g[i];
  for (int i = lane; i < na * nfl; i += 32) {
    const int r = i / nfl, c = i - r * nfl;
    send[o + na + i] = TR ? S[(int64_t)c * nfl + r] : S[i];
  }
}

// a7 accumulate: item (owned face f, remote element e, offset o): add the strip into row f's blocks and E[f]
__global__ void __launch_bounds__(256) accumulate_kernel(const AsmArgs a, const int32_t* row_ptr, const int64_t* items,
                                                         int64_t n_items, const double* recv) {
  const int lane = threadIdx.x & 31;
  const int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (it >= n_items) return;
  const int32_t f = (int32_t)items[3 * it];
  const int64_t e = items[3 * it + 1], o = items[3 * it + 2];
  const int na = a.face_ndof[f];
  int nfe = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) { const int32_t c = a.elem_face[3 * e + k]; if (c >= 0) nfe += a.face_ndof[c]; }
  double* Ef = a.E + (a.face_off[f] - a.tr0);
  for (int i = lane; i < na; i += 32) Ef[i] = Ef[i] + recv[o + i];
  const double* strip = recv + o + na;
  int soff = 0;
  for (int k = 0; k < 3; ++k) {
    const int32_t c = a.elem_face[3 * e + k];
    if (c < 0) continue;
    const int nb = a.face_ndof[c];
    int64_t q = -1;
    for (int32_t j = row_ptr[f - a.f0]; j < row_ptr[f - a.f0 + 1]; ++j)
      if (a.col_idx[j] == c) q = j;
    double* dst = a.K + a.blk_off[q];
    for (int idx = lane; idx < na * nb; idx += 32) {
      const int r = idx / nb, cc = idx - r * nb;
      dst[idx] = dst[idx] + strip[(int64_t)r * nfe + soff + cc];
    }
    soff += nb;
  }
}

__global__ void first_error_kernel(const int32_t* info, int64_t n, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (info[i] != 0) atomicMin(reinterpret_cast<unsigned long long*>(out), (unsigned long long)i);
}

AsmArgs make_args(const Plan& p, const double* S, const double* g, double* K, double* E) {
  AsmArgs a;
  a.S = S; a.g = g; a.K = K; a.E = E;
  a.elem_face = p.d_elem_face; a.face_elem = p.d_face_elem; a.face_ndof = p.d_face_ndof; a.nf = p.d_nf;
  a.face_off = p.d_face_off; a.offS = p.d_off[OFF_S]; a.offG = p.d_off[OFF_G];
  a.col_idx = p.sk.d_col_idx; a.blk_row = p.sk.d_blk_row; a.blk_off = p.sk.d_blk_off;
  a.eb = p.eb; a.n = p.n; a.nnzb = p.sk.nnzb; a.f0 = p.sk.f0; a.f1 = p.sk.f1; a.tr0 = p.sk.tr0;
  return a;
}

unsigned blocks_for(int64_t threads) { return (unsigned)((threads + 255) / 256); }

}  // namespace

cudaError_t skeleton_symbolic(Plan& p, cudaStream_t s) {
  Skeleton& k = p.sk;
  const int64_t nrows = k.f1 - k.f0;
  int64_t *cnt = nullptr, *vals = nullptr, *rs = nullptr, *vs = nullptr;
  // every allocation is checked (OOM -> the caller's HDG_ERR_NOMEM, no launch through a null pointer); the
  // temporaries are freed on every exit path, the CSR arrays by free_plan
  auto done = [&](cudaError_t e) {
    cudaFree(cnt); cudaFree(vals); cudaFree(rs); cudaFree(vs);
    return e;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&cnt, sizeof(int64_t) * (nrows + 1))) != cudaSuccess) return done(e);
  if ((e = cudaMalloc(&vals, sizeof(int64_t) * (nrows + 1))) != cudaSuccess) return done(e);
  if ((e = cudaMalloc(&rs, sizeof(int64_t) * (nrows + 1))) != cudaSuccess) return done(e);
  if ((e = cudaMalloc(&vs, sizeof(int64_t) * (nrows + 1))) != cudaSuccess) return done(e);
  if (nrows > 0)
    sym_count_kernel<<<blocks_for(nrows), 256, 0, s>>>(p.d_elem_face, p.d_face_elem, p.d_face_ndof, k.f0, nrows, cnt, vals);
  scan_kernel<<<1, 1024, 0, s>>>(cnt, nrows, rs);
  scan_kernel<<<1, 1024, 0, s>>>(vals, nrows, vs);
  int64_t tot[2];
  if ((e = cudaMemcpyAsync(&tot[0], rs + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return done(e);
  if ((e = cudaMemcpyAsync(&tot[1], vs + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return done(e);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return done(e);
  k.nnzb = tot[0];
  k.nvals = tot[1];
  if ((e = cudaMalloc(&k.d_row_ptr, sizeof(int32_t) * (nrows + 1))) != cudaSuccess) return done(e);
  if ((e = cudaMalloc(&k.d_col_idx, sizeof(int32_t) * (k.nnzb > 0 ? k.nnzb : 1))) != cudaSuccess) return done(e);
  if ((e = cudaMalloc(&k.d_blk_off, sizeof(int64_t) * (k.nnzb + 1))) != cudaSuccess) return done(e);
  if ((e = cudaMalloc(&k.d_blk_row, sizeof(int32_t) * (k.nnzb > 0 ? k.nnzb : 1))) != cudaSuccess) return done(e);
  sym_fill_kernel<<<blocks_for(nrows + 1), 256, 0, s>>>(p.d_elem_face, p.d_face_elem, p.d_face_ndof, k.f0, nrows, rs, vs,
                                                        k.d_row_ptr, k.d_col_idx, k.d_blk_off, k.d_blk_row);
  e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  return done(e);
}

cudaError_t launch_assemble(const Plan& p, const double* S, const double* g, double* K, double* E, double* send,
                            cudaStream_t s, int64_t* launches, bool transposed) {
  const AsmArgs a = make_args(p, S, g, K, E);
  if (p.sk.nnzb > 0) {
    if (transposed) assemble_kernel<true><<<blocks_for(32 * p.sk.nnzb), 256, 0, s>>>(a);
    else assemble_kernel<false><<<blocks_for(32 * p.sk.nnzb), 256, 0, s>>>(a);
    ++*launches;
  }
  if (p.sk.f1 > p.sk.f0) { assemble_rhs_kernel<<<blocks_for(32 * (p.sk.f1 - p.sk.f0)), 256, 0, s>>>(a); ++*launches; }
  if (p.sk.n_send_items > 0) {
    if (transposed) pack_kernel<true><<<blocks_for(32 * p.sk.n_send_items), 256, 0, s>>>(a, p.sk.d_send_items, p.sk.n_send_items, send);
    else pack_kernel<false><<<blocks_for(32 * p.sk.n_send_items), 256, 0, s>>>(a, p.sk.d_send_items, p.sk.n_send_items, send);
    ++*launches;
  }
  return cudaGetLastError();
}

cudaError_t launch_accumulate(const Plan& p, const double* recv, double* K, double* E, cudaStream_t s, int64_t* launches) {
  const AsmArgs a = make_args(p, nullptr, nullptr, K, E);
  if (p.sk.n_recv_items > 0) {
    accumulate_kernel<<<blocks_for(32 * p.sk.n_recv_items), 256, 0, s>>>(a, p.sk.d_row_ptr, p.sk.d_recv_items,
                                                                        p.sk.n_recv_items, recv);
    ++*launches;
  }
  return cudaGetLastError();
}

cudaError_t launch_first_error(const int32_t* info, int64_t n, int64_t* d_out, cudaStream_t s) {
  const int64_t init = INT64_MAX;
  cudaMemcpyAsync(d_out, &init, sizeof(int64_t), cudaMemcpyHostToDevice, s);
  if (n > 0) first_error_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(info, n, d_out);
  return cudaGetLastError();
}

}  // namespace hdg
