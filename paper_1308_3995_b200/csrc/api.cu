// api.cu — the C ABI of libhdg (include/hdg.h): context, plan (row a0), argument checking and dispatch of the
// condensation (a1-a5), skeleton assembly / exchange (a6-a7) and back-substitution (a8) kernels.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <tuple>

#include "hdg_internal.cuh"

using namespace hdg;

int64_t hdg::grid_cap(int64_t grid) {
  static const int64_t cap = [] {
    const char* v = getenv("HDG_MAX_GRID");
    return v ? std::max<int64_t>(1, atoll(v)) : (int64_t)0;
  }();
  return cap > 0 && grid > cap ? cap : grid;
}

namespace {

const char* kVersion = "libhdg 0.1 (sm_100a, fp64)";

hdg_status fail(hdg_ctx ctx, hdg_status st, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    ctx->last_error = buf;
  }
  return st;
}

hdg_status cuda_fail(hdg_ctx ctx, cudaError_t e, const char* where) {
  return fail(ctx, HDG_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define HDG_CUDA(ctx, call)                                    \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #call);   \
  } while (0)

template <class T>
cudaError_t upload(T** dst, const T* src, size_t n) {
  cudaError_t e = cudaMalloc(dst, sizeof(T) * (n > 0 ? n : 1));
  if (e != cudaSuccess) return e;
  if (n > 0) e = cudaMemcpy(*dst, src, sizeof(T) * n, cudaMemcpyHostToDevice);
  return e;
}

void free_plan(Plan& p) {
  cudaFree(p.d_elem_face); cudaFree(p.d_face_elem); cudaFree(p.d_face_ndof); cudaFree(p.d_face_off);
  cudaFree(p.d_ne); cudaFree(p.d_nf);
  for (auto& o : p.d_off) cudaFree(o);
  for (auto& b : p.buckets) cudaFree(b.d_elems);
  cudaFree(p.sk.d_row_ptr); cudaFree(p.sk.d_col_idx); cudaFree(p.sk.d_blk_off); cudaFree(p.sk.d_blk_row);
  cudaFree(p.sk.d_send_items); cudaFree(p.sk.d_recv_items);
  cudaFree(p.d_scratch);
  cudaFree(p.d_send); cudaFree(p.d_recv);
  cudaFree(p.d_redo); cudaFree(p.d_redo_count); cudaFree(p.d_mark);
  cudaFree(p.sw.V); cudaFree(p.sw.w); cudaFree(p.sw.z); cudaFree(p.sw.partial); cudaFree(p.sw.h); cudaFree(p.sw.Dinv);
  cudaFree(p.sw.dinv_off);
  cudaFree(p.sw.xfull); cudaFree(p.sw.hsend); cudaFree(p.sw.hrecv); cudaFree(p.sw.d_hsend_idx); cudaFree(p.sw.d_hrecv_idx);
  cudaFree(p.d_eblk); cudaFree(p.d_eE); cudaFree(p.d_eslot);
  p = Plan();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// HDG_CONDENSE_KERNEL=panel|sweep forces one condensation kernel for every bucket it supports (A/B comparisons,
// tests of both paths)
bool force_panel() {
  const char* v = getenv("HDG_CONDENSE_KERNEL");
  return v && strcmp(v, "panel") == 0;
}
bool force_sweep() {
  const char* v = getenv("HDG_CONDENSE_KERNEL");
  return v && strcmp(v, "sweep") == 0;
}

// a7 exchange layout of one rank's slab (host only, shared by hdg_plan and hdg_exchange_layout): for every face
// slot of a local element whose face row is owned by another rank (its left element is remote), one send item
// (face, local element, offset); for every owned face row whose right element is remote, one recv item (face,
// global element, offset). Items are grouped by peer rank, then face id. Each item carries the face's g slice
// and its n_fp x n_f strip of S_e: n_fp (1 + n_f) doubles.
struct ExchangeLayout {
  std::vector<int64_t> send_counts, send_displs, recv_counts, recv_displs, send_items, recv_items;
  int64_t send_doubles = 0, recv_doubles = 0;
};

void build_exchange_layout(const hdg_mesh* m, int rank, int R, ExchangeLayout& x) {
  const int64_t eb = m->elem_begin, n = m->n_elem, F = m->n_face;
  x.send_counts.assign(R, 0); x.send_displs.assign(R, 0);
  x.recv_counts.assign(R, 0); x.recv_displs.assign(R, 0);
  auto rank_of = [&](int64_t e) {
    return (int)(std::upper_bound(m->rank_elem_begin, m->rank_elem_begin + R + 1, e) - m->rank_elem_begin) - 1;
  };
  auto nf_of = [&](int64_t e) {
    int t = 0;
    for (int k = 0; k < 3; ++k) { const int32_t f = m->elem_face[3 * e + k]; if (f >= 0) t += m->face_ndof[f]; }
    return t;
  };
  std::vector<std::tuple<int, int64_t, int64_t>> snd, rcv;   // (peer, face, element)
  for (int64_t l = 0; l < n; ++l)
    for (int k = 0; k < 3; ++k) {
      const int32_t f = m->elem_face[3 * (eb + l) + k];
      if (f < 0) continue;
      const int32_t left = m->face_elem[2 * f];
      if (left < eb || left >= eb + n) snd.emplace_back(rank_of(left), f, l);
    }
  for (int64_t f = 0; f < F; ++f) {
    const int32_t left = m->face_elem[2 * f], r = m->face_elem[2 * f + 1];
    if (left >= eb && left < eb + n && r >= 0 && (r < eb || r >= eb + n)) rcv.emplace_back(rank_of(r), f, r);
  }
  (void)rank;
  std::sort(snd.begin(), snd.end());
  std::sort(rcv.begin(), rcv.end());
  int64_t o = 0;
  for (auto& t : snd) {
    const int peer = std::get<0>(t);
    const int64_t f = std::get<1>(t), l = std::get<2>(t);
    const int64_t sz = (int64_t)m->face_ndof[f] * (1 + nf_of(eb + l));
    x.send_items.insert(x.send_items.end(), {f, l, o});
    x.send_counts[peer] += sz;
    o += sz;
  }
  x.send_doubles = o;
  o = 0;
  for (auto& t : rcv) {
    const int peer = std::get<0>(t);
    const int64_t f = std::get<1>(t), e = std::get<2>(t);
    const int64_t sz = (int64_t)m->face_ndof[f] * (1 + nf_of(e));
    x.recv_items.insert(x.recv_items.end(), {f, e, o});
    x.recv_counts[peer] += sz;
    o += sz;
  }
  x.recv_doubles = o;
  for (int r = 1; r < R; ++r) {
    x.send_displs[r] = x.send_displs[r - 1] + x.send_counts[r - 1];
    x.recv_displs[r] = x.recv_displs[r - 1] + x.recv_counts[r - 1];
  }
}

// a6 (+ a7): assemble the owned rows and pack contributions to rows owned by other ranks; with an NCCL
// communicator the exchange and the ordered accumulate follow on the same stream (no host sync). Without one the
// caller transports `send` and finishes with hdg_skeleton_accumulate (the three-call protocol).
hdg_status assemble_and_exchange(hdg_ctx ctx, const double* S, const double* g, double* K, double* E, double* send,
                                 cudaStream_t s, bool transposed, const char* name) {
  const Plan& p = ctx->plan;
  const bool lib_x = ctx->nccl_comm && ctx->nranks > 1;
  double* sbuf = lib_x ? p.d_send : send;
  HDG_CUDA(ctx, launch_assemble(p, S, g, K, E, sbuf, s, &ctx->launches, transposed));
  if (lib_x) {
    std::string err;
    if (!nccl_exchange(ctx->nccl_comm, p, ctx->rank, ctx->nranks, p.d_send, p.d_recv, s, &err))
      return fail(ctx, HDG_ERR_NCCL, "%s: %s", name, err.c_str());
    HDG_CUDA(ctx, launch_accumulate(p, p.d_recv, K, E, s, &ctx->launches));
  }
  return HDG_OK;
}

}  // namespace

extern "C" {

const char* hdg_version(void) { return kVersion; }
int hdg_max_elem_ndof(void) { return kMaxNe; }
int hdg_max_face_ndof(void) { return kMaxNf; }

const char* hdg_status_string(hdg_status s) {
  switch (s) {
    case HDG_OK: return "ok";
    case HDG_ERR_ARG: return "invalid argument";
    case HDG_ERR_SINGULAR: return "singular local block";
    case HDG_ERR_CUDA: return "CUDA error";
    case HDG_ERR_NOMEM: return "out of memory";
    case HDG_ERR_STATE: return "invalid state";
    case HDG_ERR_UNSUPPORTED: return "unsupported size";
    case HDG_ERR_NCCL: return "NCCL error";
  }
  return "unknown status";
}

hdg_status hdg_get_unique_id(unsigned char id[128]) {
  if (!id) return HDG_ERR_ARG;
  std::string err;
  if (!nccl_unique_id(id, &err)) {
    std::fprintf(stderr, "hdg_get_unique_id: %s\n", err.c_str());
    return HDG_ERR_NCCL;
  }
  return HDG_OK;
}

hdg_status hdg_ctx_create(hdg_ctx* out, int device, int rank, int nranks, const unsigned char* nccl_id) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) return HDG_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return HDG_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return HDG_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return HDG_ERR_CUDA;
  if (prop.major != 10) return HDG_ERR_UNSUPPORTED;   // built for sm_100a only
  hdg_ctx c = new hdg_ctx_s;
  c->device = device;
  c->rank = rank;
  c->nranks = nranks;
  c->sms = prop.multiProcessorCount;
  c->smem_optin = prop.sharedMemPerBlockOptin;
  if (nccl_id) {
    std::string err;
    if (!nccl_comm_init(&c->nccl_comm, nranks, rank, nccl_id, &err)) {
      std::fprintf(stderr, "hdg_ctx_create: %s\n", err.c_str());
      delete c;
      return HDG_ERR_NCCL;
    }
  }
  *out = c;
  return HDG_OK;
}

int hdg_ctx_has_comm(hdg_ctx ctx) { return ctx && ctx->nccl_comm ? 1 : 0; }

void hdg_ctx_destroy(hdg_ctx ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  free_plan(ctx->plan);
  nccl_comm_destroy(ctx->nccl_comm);
  delete ctx;
}

const char* hdg_last_error(hdg_ctx ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int64_t hdg_launch_count(hdg_ctx ctx) { return ctx ? ctx->launches : 0; }

hdg_status hdg_debug_set_trace(hdg_ctx ctx, long long* trace) {
  if (!ctx) return HDG_ERR_ARG;
  ctx->trace = trace;
  return HDG_OK;
}

hdg_status hdg_plan(hdg_ctx ctx, const hdg_mesh* m, hdg_plan_info* info, hdg_stream stream) {
  if (!ctx) return HDG_ERR_ARG;
  if (!m || !info || !m->elem_face || !m->face_elem || !m->face_ndof || !m->elem_ndof)
    return fail(ctx, HDG_ERR_ARG, "hdg_plan: null mesh array");
  const int64_t E = m->n_elem_global, F = m->n_face, eb = m->elem_begin, n = m->n_elem;
  if (E < 0 || F < 0 || eb < 0 || n < 0 || eb + n > E || E > INT32_MAX || F > INT32_MAX)
    return fail(ctx, HDG_ERR_ARG, "hdg_plan: bad sizes E=%lld F=%lld begin=%lld n=%lld", (long long)E, (long long)F,
                (long long)eb, (long long)n);
  if (ctx->nranks > 1) {
    if (!m->rank_elem_begin) return fail(ctx, HDG_ERR_ARG, "hdg_plan: rank_elem_begin required for nranks > 1");
    if (m->rank_elem_begin[ctx->rank] != eb || m->rank_elem_begin[ctx->rank + 1] != eb + n ||
        m->rank_elem_begin[0] != 0 || m->rank_elem_begin[ctx->nranks] != E)
      return fail(ctx, HDG_ERR_ARG, "hdg_plan: rank_elem_begin inconsistent with elem_begin/n_elem");
    for (int r = 0; r < ctx->nranks; ++r)
      if (m->rank_elem_begin[r + 1] < m->rank_elem_begin[r])
        return fail(ctx, HDG_ERR_ARG, "hdg_plan: rank_elem_begin is not non-decreasing at rank %d", r);
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  free_plan(ctx->plan);
  Plan& p = ctx->plan;
  p.E = E; p.F = F; p.eb = eb; p.n = n;

  // ---- validate connectivity ---------------------------------------------------------------------------------
  for (int64_t f = 0; f < F; ++f) {
    const int32_t l = m->face_elem[2 * f], r = m->face_elem[2 * f + 1];
    if (l < 0 || l >= E || r >= E || (r >= 0 && r <= l))
      return fail(ctx, HDG_ERR_ARG, "hdg_plan: face %lld has bad (left,right) = (%d,%d)", (long long)f, l, r);
    const int32_t nd = m->face_ndof[f];
    if (nd <= 0 || (nd & 1)) return fail(ctx, HDG_ERR_UNSUPPORTED, "hdg_plan: face %lld trace size %d (must be even, > 0)", (long long)f, nd);
  }
  // every element's slots (remote neighbours too: the symbolic structure, the exchange layout and the
  // accumulate kernel index face_ndof / col_idx through them), and the faces' back-references
  for (int64_t e = 0; e < E; ++e)
    for (int k = 0; k < 3; ++k) {
      const int32_t f = m->elem_face[3 * e + k];
      if (f < -1 || f >= F) return fail(ctx, HDG_ERR_ARG, "hdg_plan: element %lld slot %d face %d out of range", (long long)e, k, f);
      if (f >= 0 && m->face_elem[2 * f] != e && m->face_elem[2 * f + 1] != e)
        return fail(ctx, HDG_ERR_ARG, "hdg_plan: element %lld lists face %d which does not list it", (long long)e, f);
    }
  std::vector<int64_t> face_off(F + 1, 0);
  for (int64_t f = 0; f < F; ++f) face_off[f + 1] = face_off[f] + m->face_ndof[f];
  for (int64_t f = 0; f < F; ++f) p.max_face_ndof = std::max<int>(p.max_face_ndof, m->face_ndof[f]);
  p.n_trace = face_off[F];

  std::vector<int32_t> ne(n), nf(n);
  for (int64_t l = 0; l < n; ++l) {
    const int64_t e = eb + l;
    int t = 0;
    for (int k = 0; k < 3; ++k) {
      const int32_t f = m->elem_face[3 * e + k];
      if (f < -1 || f >= F) return fail(ctx, HDG_ERR_ARG, "hdg_plan: element %lld slot %d face %d out of range", (long long)e, k, f);
      if (f >= 0) {
        if (m->face_elem[2 * f] != e && m->face_elem[2 * f + 1] != e)
          return fail(ctx, HDG_ERR_ARG, "hdg_plan: element %lld lists face %d which does not list it", (long long)e, f);
        t += m->face_ndof[f];
      }
    }
    ne[l] = m->elem_ndof[e];
    nf[l] = t;
    if (ne[l] <= 0 || (ne[l] & 3)) return fail(ctx, HDG_ERR_UNSUPPORTED, "hdg_plan: element %lld n_e=%d (must be a positive multiple of 4)", (long long)e, ne[l]);
    if (ne[l] > kMaxNe || nf[l] > kMaxNf)
      return fail(ctx, HDG_ERR_UNSUPPORTED, "hdg_plan: element %lld n_e=%d n_f=%d exceeds %d/%d", (long long)e, ne[l], nf[l], kMaxNe, kMaxNf);
    p.max_ne = std::max(p.max_ne, ne[l]);
    p.max_nf = std::max(p.max_nf, nf[l]);
  }

  // ---- packed offsets --------------------------------------------------------------------------------------------
  std::vector<std::vector<int64_t>> off(N_OFF, std::vector<int64_t>(n + 1, 0));
  for (int64_t l = 0; l < n; ++l) {
    const int64_t a = ne[l], f = nf[l];
    const int64_t sz[N_OFF] = {a * a, a * f, f * a, f * f, a, f, f * f, f, a, factor_bytes((int)a), a * (f + 1)};
    for (int k = 0; k < N_OFF; ++k) off[k][l + 1] = off[k][l] + sz[k];
  }
  p.len.resize(N_OFF);
  for (int k = 0; k < N_OFF; ++k) p.len[k] = off[k][n];

  // ---- buckets by (n_e, n_f), heaviest first ------------------------------------------------------------------
  std::map<std::pair<int, int>, std::vector<int32_t>> bk;
  for (int64_t l = 0; l < n; ++l) bk[{ne[l], nf[l]}].push_back((int32_t)l);
  std::vector<std::pair<std::pair<int, int>, std::vector<int32_t>>> order(bk.begin(), bk.end());
  std::sort(order.begin(), order.end(), [](const auto& x, const auto& y) {
    const double wx = (double)x.first.first * x.first.first * (x.first.first + 3.0 * x.first.second) * x.second.size();
    const double wy = (double)y.first.first * y.first.first * (y.first.first + 3.0 * y.first.second) * y.second.size();
    return wx > wy;
  });
  int64_t scratch = 0;
  for (auto& b : order) {
    Bucket B;
    B.ne = b.first.first;
    B.nf = b.first.second;
    B.count = (int64_t)b.second.size();
    const Geo geo(B.ne, B.nf);
    B.t_in_smem = geo.smem_bytes(true) <= (int64_t)ctx->smem_optin;
    // measured on the box: the sweep kernel (chain warp + MMA workers; 2 CTAs per SM when they fit) wins for
    // n_e >= 96 (C4: 45 vs 57 ms), for C5's n_e = 72 buckets (C5 slab 85.0 -> 81.6 ms vs the panel kernel) and
    // n_e <= 32 (C2: 0.82 vs 0.95 ms); the panel kernel for n_e = 60 (C3: 34 vs 40 ms). The (120, n_f > 48)
    // buckets, whose C rows do not fit beside T, stay on the panel kernel (the GT sweep measured 85.0 -> 87.5 ms)
    const char* forced = getenv("HDG_CONDENSE_KERNEL");
    const std::string fk = forced ? forced : "";
    // small elements (C1, C2): one warp per element, 16+ elements in flight per SM (C2: 0.71 ms on the sweep
    // kernel, see DESIGN §11 for the warp kernel's number); HDG_CONDENSE_KERNEL=sweep|panel force the others
    B.warp = warp_supported(B.ne, B.nf) && fk != "sweep" && fk != "panel";
    const int sweep_min = getenv("HDG_SWEEP_MIN_NE") ? atoi(getenv("HDG_SWEEP_MIN_NE")) : 64;   // experiments
    B.sweep = !B.warp && sweep_supported(B.ne, B.nf, ctx->smem_optin) && fk != "panel" &&
              (B.ne >= sweep_min || B.ne <= 32 || fk == "sweep");
    // the row-tile kernel (condense_rows.cu): HDG_CONDENSE_KERNEL=rows
    B.rows = !B.warp && fk == "rows" && rows_supported(B.ne, B.nf, ctx->smem_optin);
    if (B.rows) B.sweep = false;
    // elements larger than one SM (C5's n_e = 180, 252): the sweep kernel on an L2-resident global slab
    B.sweep_gt = !B.warp && !B.sweep && !B.rows && !B.t_in_smem && fk != "panel" && sweep_gt_supported(B.ne, B.nf);
    if (!B.warp && !B.sweep && !B.sweep_gt && !B.rows && !B.t_in_smem) scratch = std::max(scratch, geo.t_doubles() * ctx->sms);
    if (B.sweep || B.sweep_gt || B.rows) {   // exact-path (and GT working) slab per resident CTA (at most 2 per SM)
      const SweepGeo sg(B.ne, B.nf);
      scratch = std::max(scratch, ((int64_t)sg.RA * sg.ldT + (int64_t)sg.NF8 * sg.ldC) * 2 * ctx->sms);
    }
    HDG_CUDA(ctx, upload(&B.d_elems, b.second.data(), b.second.size()));
    p.buckets.push_back(B);
  }
  if (scratch > 0) {
    if (cudaMalloc(&p.d_scratch, sizeof(double) * scratch) != cudaSuccess)
      return fail(ctx, HDG_ERR_NOMEM, "hdg_plan: scratch of %lld doubles", (long long)scratch);
    p.scratch_doubles = scratch;
  }
  if (std::any_of(p.buckets.begin(), p.buckets.end(), [](const Bucket& b) { return b.rows; })) {
    if (cudaMalloc(&p.d_redo, sizeof(int32_t) * std::max<int64_t>(1, n)) != cudaSuccess ||
        cudaMalloc(&p.d_redo_count, sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&p.d_mark, sizeof(int32_t) * std::max<int64_t>(1, n)) != cudaSuccess)
      return fail(ctx, HDG_ERR_NOMEM, "hdg_plan: redo list");
    HDG_CUDA(ctx, cudaMemset(p.d_mark, 0, sizeof(int32_t) * std::max<int64_t>(1, n)));
  }

  // ---- owned skeleton rows ---------------------------------------------------------------------------------------
  int64_t fmin = F, fmax = -1, cnt = 0;
  for (int64_t f = 0; f < F; ++f) {
    const int32_t l = m->face_elem[2 * f];
    if (l >= eb && l < eb + n) { fmin = std::min(fmin, f); fmax = std::max(fmax, f); ++cnt; }
  }
  if (cnt == 0) { fmin = 0; fmax = -1; }
  if (cnt != fmax - fmin + 1) return fail(ctx, HDG_ERR_ARG, "hdg_plan: owned faces are not a contiguous id range");
  p.sk.f0 = fmin;
  p.sk.f1 = fmax + 1;
  p.sk.tr0 = face_off[p.sk.f0];
  p.sk.ntr = face_off[p.sk.f1] - face_off[p.sk.f0];

  // ---- uploads ----------------------------------------------------------------------------------------------------
  HDG_CUDA(ctx, upload(&p.d_elem_face, m->elem_face, (size_t)(3 * E)));
  HDG_CUDA(ctx, upload(&p.d_face_elem, m->face_elem, (size_t)(2 * F)));
  HDG_CUDA(ctx, upload(&p.d_face_ndof, m->face_ndof, (size_t)F));
  HDG_CUDA(ctx, upload(&p.d_face_off, face_off.data(), (size_t)(F + 1)));
  HDG_CUDA(ctx, upload(&p.d_ne, ne.data(), (size_t)n));
  HDG_CUDA(ctx, upload(&p.d_nf, nf.data(), (size_t)n));
  for (int k = 0; k < N_OFF; ++k) HDG_CUDA(ctx, upload(&p.d_off[k], off[k].data(), (size_t)(n + 1)));
  {
    const cudaError_t e = skeleton_symbolic(p, s);
    if (e == cudaErrorMemoryAllocation) return fail(ctx, HDG_ERR_NOMEM, "hdg_plan: block-CSR structure: %s", cudaGetErrorString(e));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "hdg_plan: skeleton_symbolic");
  }

  // ---- exchange lists (faces shared between slabs) ----------------------------------------------------------------
  const int R = ctx->nranks;
  if (R > 1) {
    ExchangeLayout x;
    build_exchange_layout(m, ctx->rank, R, x);
    p.sk.send_counts = x.send_counts; p.sk.send_displs = x.send_displs;
    p.sk.recv_counts = x.recv_counts; p.sk.recv_displs = x.recv_displs;
    p.sk.send_doubles = x.send_doubles; p.sk.recv_doubles = x.recv_doubles;
    p.sk.n_send_items = (int64_t)x.send_items.size() / 3;
    p.sk.n_recv_items = (int64_t)x.recv_items.size() / 3;
    HDG_CUDA(ctx, upload(&p.sk.d_send_items, x.send_items.data(), x.send_items.size()));
    HDG_CUDA(ctx, upload(&p.sk.d_recv_items, x.recv_items.data(), x.recv_items.size()));
    // ---- halo lists of the distributed skeleton solve: the columns of my owned rows owned elsewhere (received
    //      before every SpMV), and my owned faces in the rows of others (sent); the adjacency is symmetric (two
    //      faces couple iff they share an element), so both lists follow from my rows alone
    {
      auto rank_of = [&](int64_t e) {
        return (int)(std::upper_bound(m->rank_elem_begin, m->rank_elem_begin + R + 1, e) - m->rank_elem_begin) - 1;
      };
      std::vector<int> fown(F);
      p.rank_tr0.assign(R, 0);
      p.rank_ntr.assign(R, 0);
      std::vector<int64_t> fmin_r(R, F), fmax_r(R, -1);
      for (int64_t f = 0; f < F; ++f) {
        fown[f] = rank_of(m->face_elem[2 * f]);
        fmin_r[fown[f]] = std::min(fmin_r[fown[f]], f);
        fmax_r[fown[f]] = std::max(fmax_r[fown[f]], f);
      }
      for (int r = 0; r < R; ++r)
        if (fmax_r[r] >= 0) {
          p.rank_tr0[r] = face_off[fmin_r[r]];
          p.rank_ntr[r] = face_off[fmax_r[r] + 1] - face_off[fmin_r[r]];
        }
      std::vector<std::set<int32_t>> sendf(R), recvf(R);
      for (int64_t f = p.sk.f0; f < p.sk.f1; ++f)
        for (int side = 0; side < 2; ++side) {
          const int32_t e = m->face_elem[2 * f + side];
          if (e < 0) continue;
          for (int kk = 0; kk < 3; ++kk) {
            const int32_t c = m->elem_face[3 * e + kk];
            if (c < 0 || fown[c] == ctx->rank) continue;
            recvf[fown[c]].insert(c);
            sendf[fown[c]].insert((int32_t)f);
          }
        }
      p.halo_scnt.assign(R, 0); p.halo_sdsp.assign(R, 0); p.halo_rcnt.assign(R, 0); p.halo_rdsp.assign(R, 0);
      p.halo_send_idx.clear(); p.halo_recv_idx.clear();
      for (int r = 0; r < R; ++r) {
        p.halo_sdsp[r] = (int64_t)p.halo_send_idx.size();
        for (int32_t f : sendf[r])
          for (int64_t d = face_off[f]; d < face_off[f + 1]; ++d) p.halo_send_idx.push_back(d);
        p.halo_scnt[r] = (int64_t)p.halo_send_idx.size() - p.halo_sdsp[r];
        p.halo_rdsp[r] = (int64_t)p.halo_recv_idx.size();
        for (int32_t f : recvf[r])
          for (int64_t d = face_off[f]; d < face_off[f + 1]; ++d) p.halo_recv_idx.push_back(d);
        p.halo_rcnt[r] = (int64_t)p.halo_recv_idx.size() - p.halo_rdsp[r];
      }
    }
    if (ctx->nccl_comm) {   // the library owns the exchange buffers (a7 runs inside hdg_assemble_*)
      if (cudaMalloc(&p.d_send, sizeof(double) * std::max<int64_t>(1, x.send_doubles)) != cudaSuccess ||
          cudaMalloc(&p.d_recv, sizeof(double) * std::max<int64_t>(1, x.recv_doubles)) != cudaSuccess)
        return fail(ctx, HDG_ERR_NOMEM, "hdg_plan: exchange buffers");
    }
  } else {
    p.sk.send_counts.assign(1, 0); p.sk.send_displs.assign(1, 0);
    p.sk.recv_counts.assign(1, 0); p.sk.recv_displs.assign(1, 0);
  }

  p.valid = true;
  std::memset(info, 0, sizeof *info);
  info->n_elem = n;
  info->len_A = p.len[OFF_A]; info->len_B = p.len[OFF_B]; info->len_C = p.len[OFF_C]; info->len_D = p.len[OFF_D];
  info->len_re = p.len[OFF_RE]; info->len_rf = p.len[OFF_RF];
  info->len_S = p.len[OFF_S]; info->len_g = p.len[OFF_G]; info->len_u = p.len[OFF_U];
  info->factor_bytes = p.len[OFF_F];
  info->owned_face_begin = p.sk.f0; info->n_owned_faces = p.sk.f1 - p.sk.f0;
  info->nnzb = p.sk.nnzb; info->nvals = p.sk.nvals;
  info->owned_trace_begin = p.sk.tr0; info->n_owned_trace = p.sk.ntr;
  info->n_trace = p.n_trace;
  info->n_buckets = (int32_t)p.buckets.size();
  info->max_ne = p.max_ne; info->max_nf = p.max_nf;
  info->send_doubles = p.sk.send_doubles; info->recv_doubles = p.sk.recv_doubles;
  info->len_X = p.len[OFF_X];
  return HDG_OK;
}

// fused condense -> assemble tables (per local element: the K offset of each of its 3 x 3 slot-pair blocks, the E
// offset of each slot, the slot start rows), built once per plan from the block-CSR structure
static hdg_status build_fused_tables(hdg_ctx ctx) {
  Plan& p = ctx->plan;
  if (p.d_eblk) return HDG_OK;
  const Skeleton& k = p.sk;
  const int64_t nrows = k.f1 - k.f0, n = p.n;
  std::vector<int32_t> rp(nrows + 1), ci(std::max<int64_t>(k.nnzb, 1)), ef(3 * p.E), fnd(p.F);
  std::vector<int64_t> bo(k.nnzb + 1), fo(p.F + 1);
  HDG_CUDA(ctx, cudaMemcpy(rp.data(), k.d_row_ptr, sizeof(int32_t) * (nrows + 1), cudaMemcpyDeviceToHost));
  if (k.nnzb) HDG_CUDA(ctx, cudaMemcpy(ci.data(), k.d_col_idx, sizeof(int32_t) * k.nnzb, cudaMemcpyDeviceToHost));
  HDG_CUDA(ctx, cudaMemcpy(bo.data(), k.d_blk_off, sizeof(int64_t) * (k.nnzb + 1), cudaMemcpyDeviceToHost));
  HDG_CUDA(ctx, cudaMemcpy(ef.data(), p.d_elem_face, sizeof(int32_t) * 3 * p.E, cudaMemcpyDeviceToHost));
  HDG_CUDA(ctx, cudaMemcpy(fnd.data(), p.d_face_ndof, sizeof(int32_t) * p.F, cudaMemcpyDeviceToHost));
  HDG_CUDA(ctx, cudaMemcpy(fo.data(), p.d_face_off, sizeof(int64_t) * (p.F + 1), cudaMemcpyDeviceToHost));
  std::vector<int64_t> eblk(9 * std::max<int64_t>(n, 1), -1), eE(3 * std::max<int64_t>(n, 1), -1);
  std::vector<int32_t> eslot(4 * std::max<int64_t>(n, 1), 0);
  for (int64_t l = 0; l < n; ++l) {
    const int32_t* f = ef.data() + 3 * (p.eb + l);
    int32_t* so = eslot.data() + 4 * l;
    for (int a = 0; a < 3; ++a) so[a + 1] = so[a] + (f[a] >= 0 ? fnd[f[a]] : 0);
    for (int a = 0; a < 3; ++a) {
      if (f[a] < 0 || f[a] < k.f0 || f[a] >= k.f1) continue;   // no trace, or a row owned by another rank
      eE[3 * l + a] = fo[f[a]] - k.tr0;
      const int64_t r = f[a] - k.f0;
      for (int b = 0; b < 3; ++b) {
        if (f[b] < 0) continue;
        for (int q = rp[r]; q < rp[r + 1]; ++q)
          if (ci[q] == f[b]) { eblk[9 * l + 3 * a + b] = bo[q]; break; }
      }
    }
  }
  HDG_CUDA(ctx, upload(&p.d_eblk, eblk.data(), eblk.size()));
  HDG_CUDA(ctx, upload(&p.d_eE, eE.data(), eE.size()));
  HDG_CUDA(ctx, upload(&p.d_eslot, eslot.data(), eslot.size()));
  return HDG_OK;
}

static hdg_status condense_impl(hdg_ctx ctx, const double* A, const double* B, const double* C, const double* D,
                                const double* r_e, const double* r_f, const double* shift, double* S, double* g,
                                void* factors, int32_t* info, hdg_stream stream, const char* name,
                                double* X = nullptr, double* Kf = nullptr, double* Ef = nullptr) {
  if (!ctx) return HDG_ERR_ARG;
  const Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "%s: no plan", name);
  ctx->launches = 0;
  if (p.n == 0) return HDG_OK;
  const void* ptrs[] = {A, B, C, D, r_e, r_f, Kf ? (const void*)Kf : S, Kf ? (const void*)Ef : g, factors, info};
  for (const void* q : ptrs)
    if (!q || !aligned16(q)) return fail(ctx, HDG_ERR_ARG, "%s: null or misaligned (16 B) pointer", name);
  if (shift && !aligned16(shift)) return fail(ctx, HDG_ERR_ARG, "%s: misaligned (16 B) shift", name);
  if (X && !aligned16(X)) return fail(ctx, HDG_ERR_ARG, "%s: misaligned (16 B) X", name);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  for (const Bucket& b : p.buckets) {
    CondenseArgs a;
    a.A = A; a.B = B; a.C = C; a.D = D; a.re = r_e; a.rf = r_f; a.S = S; a.g = g;
    a.shift = shift;
    a.Kf = Kf; a.Ef = Ef; a.eblk = p.d_eblk; a.eE = p.d_eE; a.eslot = p.d_eslot;
    a.factors = static_cast<unsigned char*>(factors);
    a.info = info;
    a.elems = b.d_elems;
    a.offA = p.d_off[OFF_A]; a.offB = p.d_off[OFF_B]; a.offC = p.d_off[OFF_C]; a.offD = p.d_off[OFF_D];
    a.offRe = p.d_off[OFF_RE]; a.offRf = p.d_off[OFF_RF]; a.offS = p.d_off[OFF_S]; a.offG = p.d_off[OFF_G];
    a.offF = p.d_off[OFF_F];
    a.ne = b.ne; a.nf = b.nf; a.count = b.count;
    a.scratch = p.d_scratch;
    a.trace = ctx->trace;
    a.debug = getenv("HDG_DEBUG_MODE") ? atoi(getenv("HDG_DEBUG_MODE")) : 0;
    a.redo = p.d_redo; a.redo_count = p.d_redo_count; a.mark = p.d_mark;
    // saved solutions: the warp and panel kernels form X and write it; the others get the save pass from the factors
    const bool forms_x = b.warp || (!b.rows && !b.sweep && !b.sweep_gt);
    a.Xout = (X && forms_x) ? X : nullptr;
    a.offX = p.d_off[OFF_X];
    // diagnostics: HDG_BUCKET_TIMES=1 prints each bucket's kernel time (synchronizes; never in a timed run)
    static const bool bucket_times = getenv("HDG_BUCKET_TIMES") != nullptr;
    cudaEvent_t bt0 = nullptr, bt1 = nullptr;
    if (bucket_times) {
      cudaEventCreate(&bt0);
      cudaEventCreate(&bt1);
      cudaEventRecord(bt0, s);
    }
    if (b.warp) HDG_CUDA(ctx, launch_condense_warp(a, ctx->sms, s, &ctx->launches));
    else if (b.rows) HDG_CUDA(ctx, launch_condense_rows(a, ctx->sms, ctx->smem_optin, s, &ctx->launches));
    else if (b.sweep) HDG_CUDA(ctx, launch_condense_sweep(a, ctx->sms, ctx->smem_optin, s, &ctx->launches));
    else if (b.sweep_gt) HDG_CUDA(ctx, launch_condense_sweep_gt(a, ctx->sms, s, &ctx->launches));
    else HDG_CUDA(ctx, launch_condense(a, b.t_in_smem, ctx->sms, s, &ctx->launches));
    if (bucket_times) {
      float ms = 0.f;
      cudaEventRecord(bt1, s);
      cudaEventSynchronize(bt1);
      cudaEventElapsedTime(&ms, bt0, bt1);
      fprintf(stderr, "HDG_BUCKET_TIMES ne %d nf %d count %lld kernel %s ms %.3f\n", b.ne, b.nf, (long long)b.count,
              b.warp ? "warp" : b.rows ? "rows" : b.sweep ? "sweep" : b.sweep_gt ? "sweep_gt" : "panel", ms);
      cudaEventDestroy(bt0);
      cudaEventDestroy(bt1);
    }
    if (X && !forms_x) {
      SolutionsArgs q{};
      q.factors = a.factors; q.B = B; q.re = r_e; q.X = X;
      q.elems = b.d_elems;
      q.offB = p.d_off[OFF_B]; q.offRe = p.d_off[OFF_RE]; q.offF = p.d_off[OFF_F]; q.offX = p.d_off[OFF_X];
      q.ne = b.ne; q.nf = b.nf; q.count = b.count;
      HDG_CUDA(ctx, launch_save_solutions(q, ctx->sms, s, &ctx->launches));
    }
  }
  return HDG_OK;
}

hdg_status hdg_condense(hdg_ctx ctx, const double* A, const double* B, const double* C, const double* D,
                        const double* r_e, const double* r_f, double* S, double* g, void* factors, int32_t* info,
                        hdg_stream stream) {
  return condense_impl(ctx, A, B, C, D, r_e, r_f, nullptr, S, g, factors, info, stream, "hdg_condense");
}

hdg_status hdg_condense_assemble(hdg_ctx ctx, const double* A, const double* B, const double* C, const double* D,
                                 const double* r_e, const double* r_f, double* K, double* E, void* factors,
                                 int32_t* info, hdg_stream stream) {
  if (!ctx) return HDG_ERR_ARG;
  Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "hdg_condense_assemble: no plan");
  if (ctx->nranks != 1)
    return fail(ctx, HDG_ERR_UNSUPPORTED, "hdg_condense_assemble: single rank (shared-face rows need the exchange)");
  if ((p.sk.nvals > 0 && !K) || (p.sk.ntr > 0 && !E)) return fail(ctx, HDG_ERR_ARG, "hdg_condense_assemble: null K/E");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  const hdg_status st = build_fused_tables(ctx);
  if (st != HDG_OK) return st;
  if (p.sk.nvals > 0) HDG_CUDA(ctx, cudaMemsetAsync(K, 0, sizeof(double) * p.sk.nvals, s));
  if (p.sk.ntr > 0) HDG_CUDA(ctx, cudaMemsetAsync(E, 0, sizeof(double) * p.sk.ntr, s));
  if (p.n == 0) return HDG_OK;
  return condense_impl(ctx, A, B, C, D, r_e, r_f, nullptr, nullptr, nullptr, factors, info, stream,
                       "hdg_condense_assemble", nullptr, K, E);
}

hdg_status hdg_skeleton_structure(hdg_ctx ctx, int32_t* row_ptr, int32_t* col_idx, int64_t* blk_off,
                                  hdg_stream stream) {
  if (!ctx) return HDG_ERR_ARG;
  const Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "hdg_skeleton_structure: no plan");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  const int64_t nrows = p.sk.f1 - p.sk.f0;
  if (row_ptr) HDG_CUDA(ctx, cudaMemcpyAsync(row_ptr, p.sk.d_row_ptr, sizeof(int32_t) * (nrows + 1), cudaMemcpyDeviceToDevice, s));
  if (col_idx && p.sk.nnzb) HDG_CUDA(ctx, cudaMemcpyAsync(col_idx, p.sk.d_col_idx, sizeof(int32_t) * p.sk.nnzb, cudaMemcpyDeviceToDevice, s));
  if (blk_off) HDG_CUDA(ctx, cudaMemcpyAsync(blk_off, p.sk.d_blk_off, sizeof(int64_t) * (p.sk.nnzb + 1), cudaMemcpyDeviceToDevice, s));
  return HDG_OK;
}

hdg_status hdg_condense_saved(hdg_ctx ctx, const double* A, const double* B, const double* C, const double* D,
                              const double* r_e, const double* r_f, double* S, double* g, void* factors, double* X,
                              int32_t* info, hdg_stream stream) {
  if (ctx && ctx->plan.valid && ctx->plan.n > 0 && !X) return fail(ctx, HDG_ERR_ARG, "hdg_condense_saved: null X");
  return condense_impl(ctx, A, B, C, D, r_e, r_f, nullptr, S, g, factors, info, stream, "hdg_condense_saved", X);
}

hdg_status hdg_condense_shifted(hdg_ctx ctx, const double* A, const double* B, const double* C, const double* D,
                                const double* r_e, const double* r_f, const double* shift, double* S, double* g,
                                void* factors, int32_t* info, hdg_stream stream) {
  return condense_impl(ctx, A, B, C, D, r_e, r_f, shift, S, g, factors, info, stream, "hdg_condense_shifted");
}

hdg_status hdg_assemble_skeleton(hdg_ctx ctx, const double* S, const double* g, int32_t* row_ptr, int32_t* col_idx,
                                 int64_t* blk_off, double* K, double* E, double* send, hdg_stream stream) {
  if (!ctx) return HDG_ERR_ARG;
  const Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "hdg_assemble_skeleton: no plan");
  ctx->launches = 0;
  if ((p.sk.nvals > 0 && !K) || (p.sk.ntr > 0 && !E) || (p.n > 0 && (!S || !g)))
    return fail(ctx, HDG_ERR_ARG, "hdg_assemble_skeleton: null pointer");
  if (p.sk.send_doubles > 0 && !send && !ctx->nccl_comm)
    return fail(ctx, HDG_ERR_ARG, "hdg_assemble_skeleton: send buffer required");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  const int64_t nrows = p.sk.f1 - p.sk.f0;
  if (row_ptr) HDG_CUDA(ctx, cudaMemcpyAsync(row_ptr, p.sk.d_row_ptr, sizeof(int32_t) * (nrows + 1), cudaMemcpyDeviceToDevice, s));
  if (col_idx && p.sk.nnzb) HDG_CUDA(ctx, cudaMemcpyAsync(col_idx, p.sk.d_col_idx, sizeof(int32_t) * p.sk.nnzb, cudaMemcpyDeviceToDevice, s));
  if (blk_off) HDG_CUDA(ctx, cudaMemcpyAsync(blk_off, p.sk.d_blk_off, sizeof(int64_t) * (p.sk.nnzb + 1), cudaMemcpyDeviceToDevice, s));
  return assemble_and_exchange(ctx, S, g, K, E, send, s, false, "hdg_assemble_skeleton");
}

hdg_status hdg_exchange_counts(hdg_ctx ctx, int64_t* send_counts, int64_t* send_displs, int64_t* recv_counts,
                               int64_t* recv_displs) {
  if (!ctx) return HDG_ERR_ARG;
  const Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "hdg_exchange_counts: no plan");
  for (int r = 0; r < ctx->nranks; ++r) {
    if (send_counts) send_counts[r] = p.sk.send_counts[r];
    if (send_displs) send_displs[r] = p.sk.send_displs[r];
    if (recv_counts) recv_counts[r] = p.sk.recv_counts[r];
    if (recv_displs) recv_displs[r] = p.sk.recv_displs[r];
  }
  return HDG_OK;
}

hdg_status hdg_skeleton_accumulate(hdg_ctx ctx, const double* recv, double* K, double* E, hdg_stream stream) {
  if (!ctx) return HDG_ERR_ARG;
  const Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "hdg_skeleton_accumulate: no plan");
  if (p.sk.recv_doubles > 0 && (!recv || !K || !E)) return fail(ctx, HDG_ERR_ARG, "hdg_skeleton_accumulate: null pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  HDG_CUDA(ctx, launch_accumulate(p, recv, K, E, s, &ctx->launches));
  return HDG_OK;
}

hdg_status hdg_backsubstitute(hdg_ctx ctx, const void* factors, const double* B, const double* r_e, const double* lambda,
                              double* u, hdg_stream stream) {
  if (!ctx) return HDG_ERR_ARG;
  const Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "hdg_backsubstitute: no plan");
  ctx->launches = 0;
  if (p.n == 0) return HDG_OK;
  const void* ptrs[] = {factors, B, r_e, u};
  for (const void* q : ptrs)
    if (!q || !aligned16(q)) return fail(ctx, HDG_ERR_ARG, "hdg_backsubstitute: null or misaligned (16 B) pointer");
  if (!lambda && p.n_trace > 0) return fail(ctx, HDG_ERR_ARG, "hdg_backsubstitute: null lambda");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  for (const Bucket& b : p.buckets) {
    BacksubArgs a;
    a.factors = static_cast<const unsigned char*>(factors);
    a.B = B; a.re = r_e; a.lambda = lambda; a.u = u;
    a.elems = b.d_elems;
    a.offB = p.d_off[OFF_B]; a.offRe = p.d_off[OFF_RE]; a.offU = p.d_off[OFF_U]; a.offF = p.d_off[OFF_F];
    a.elem_face = p.d_elem_face; a.face_ndof = p.d_face_ndof; a.face_off = p.d_face_off;
    a.elem_begin = p.eb;
    a.ne = b.ne; a.nf = b.nf; a.count = b.count;
    HDG_CUDA(ctx, launch_backsub(a, ctx->sms, s, &ctx->launches));
  }
  return HDG_OK;
}

// ---- adjoint (transposed) path: SURVEY.md §8(f) NEXT #1, PAPER.md:414-436 ---------------------------------------
static hdg_status adjoint_elementwise(hdg_ctx ctx, int mode, const char* name, const void* factors, const double* M,
                                      const double* rt_e, const double* rt_f, const double* lambda_t, double* out,
                                      hdg_stream stream) {
  if (!ctx) return HDG_ERR_ARG;
  const Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "%s: no plan", name);
  ctx->launches = 0;
  if (p.n == 0) return HDG_OK;
  const void* ptrs[] = {factors, M, rt_e, out};
  for (const void* q : ptrs)
    if (!q || !aligned16(q)) return fail(ctx, HDG_ERR_ARG, "%s: null or misaligned (16 B) pointer", name);
  if (mode == 1 && !lambda_t && p.n_trace > 0) return fail(ctx, HDG_ERR_ARG, "%s: null lambda_t", name);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  for (const Bucket& b : p.buckets) {
    AdjointArgs a;
    a.factors = static_cast<const unsigned char*>(factors);
    a.re = rt_e; a.rf = rt_f; a.M = M; a.lambda = lambda_t; a.out = out;
    a.elems = b.d_elems;
    a.offF = p.d_off[OFF_F]; a.offRe = p.d_off[OFF_RE]; a.offRf = p.d_off[OFF_RF];
    a.offM = p.d_off[mode == 0 ? OFF_B : OFF_C];
    a.offOut = p.d_off[mode == 0 ? OFF_G : OFF_U];
    a.elem_face = p.d_elem_face; a.face_ndof = p.d_face_ndof; a.face_off = p.d_face_off;
    a.elem_begin = p.eb;
    a.ne = b.ne; a.nf = b.nf; a.count = b.count;
    HDG_CUDA(ctx, launch_adjoint(a, mode, ctx->sms, s, &ctx->launches));
  }
  return HDG_OK;
}

hdg_status hdg_condense_adjoint_rhs(hdg_ctx ctx, const void* factors, const double* B, const double* rt_e,
                                    const double* rt_f, double* gt, hdg_stream stream) {
  if (rt_f && !aligned16(rt_f)) return fail(ctx, HDG_ERR_ARG, "hdg_condense_adjoint_rhs: misaligned rt_f");
  return adjoint_elementwise(ctx, 0, "hdg_condense_adjoint_rhs", factors, B, rt_e, rt_f, nullptr, gt, stream);
}

hdg_status hdg_backsubstitute_adjoint(hdg_ctx ctx, const void* factors, const double* C, const double* rt_e,
                                      const double* lambda_t, double* ut, hdg_stream stream) {
  return adjoint_elementwise(ctx, 1, "hdg_backsubstitute_adjoint", factors, C, rt_e, nullptr, lambda_t, ut, stream);
}

hdg_status hdg_assemble_adjoint(hdg_ctx ctx, const double* S, const double* gt, double* Kt, double* Et,
                                double* send, hdg_stream stream) {
  if (!ctx) return HDG_ERR_ARG;
  const Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "hdg_assemble_adjoint: no plan");
  ctx->launches = 0;
  if ((p.sk.nvals > 0 && !Kt) || (p.sk.ntr > 0 && !Et) || (p.n > 0 && (!S || !gt)))
    return fail(ctx, HDG_ERR_ARG, "hdg_assemble_adjoint: null pointer");
  if (p.sk.send_doubles > 0 && !send && !ctx->nccl_comm)
    return fail(ctx, HDG_ERR_ARG, "hdg_assemble_adjoint: send buffer required");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  return assemble_and_exchange(ctx, S, gt, Kt, Et, send, s, true, "hdg_assemble_adjoint");
}

hdg_status hdg_first_error(hdg_ctx ctx, const int32_t* info, int64_t* elem, int32_t* code, hdg_stream stream) {
  if (!ctx || !elem || !code) return HDG_ERR_ARG;
  const Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "hdg_first_error: no plan");
  *elem = -1;
  *code = 0;
  if (p.n == 0) return HDG_OK;
  if (!info) return fail(ctx, HDG_ERR_ARG, "hdg_first_error: null info");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  int64_t* d = nullptr;
  HDG_CUDA(ctx, cudaMalloc(&d, sizeof(int64_t)));
  int64_t h = INT64_MAX;
  cudaError_t e = launch_first_error(info, p.n, d, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "hdg_first_error");
  if (h == INT64_MAX) return HDG_OK;
  *elem = h;
  if (cudaMemcpy(code, info + h, sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(ctx, HDG_ERR_CUDA, "hdg_first_error: copy");
  return fail(ctx, HDG_ERR_SINGULAR, "singular local block: element %lld (info %d)", (long long)(p.eb + h), *code);
}

hdg_status hdg_exchange_layout(const hdg_mesh* m, int rank, int nranks, int64_t* send_counts, int64_t* send_displs,
                               int64_t* recv_counts, int64_t* recv_displs, int64_t* n_send_items, int64_t* send_items,
                               int64_t* n_recv_items, int64_t* recv_items) {
  if (!m || !m->elem_face || !m->face_elem || !m->face_ndof || !m->rank_elem_begin || nranks < 1 || rank < 0 ||
      rank >= nranks || !n_send_items || !n_recv_items)
    return HDG_ERR_ARG;
  if (m->rank_elem_begin[rank] != m->elem_begin || m->rank_elem_begin[rank + 1] != m->elem_begin + m->n_elem)
    return HDG_ERR_ARG;
  const int64_t E = m->n_elem_global, F = m->n_face;
  if (m->rank_elem_begin[0] != 0 || m->rank_elem_begin[nranks] != E) return HDG_ERR_ARG;
  for (int r = 0; r < nranks; ++r)
    if (m->rank_elem_begin[r + 1] < m->rank_elem_begin[r]) return HDG_ERR_ARG;
  for (int64_t i = 0; i < 3 * E; ++i)
    if (m->elem_face[i] < -1 || m->elem_face[i] >= F) return HDG_ERR_ARG;
  for (int64_t f = 0; f < F; ++f) {
    const int32_t l = m->face_elem[2 * f], r = m->face_elem[2 * f + 1];
    if (l < 0 || l >= E || r >= E || (r >= 0 && r <= l) || m->face_ndof[f] <= 0) return HDG_ERR_ARG;
  }
  ExchangeLayout x;
  build_exchange_layout(m, rank, nranks, x);
  for (int r = 0; r < nranks; ++r) {
    if (send_counts) send_counts[r] = x.send_counts[r];
    if (send_displs) send_displs[r] = x.send_displs[r];
    if (recv_counts) recv_counts[r] = x.recv_counts[r];
    if (recv_displs) recv_displs[r] = x.recv_displs[r];
  }
  const int64_t ns = (int64_t)x.send_items.size() / 3, nr = (int64_t)x.recv_items.size() / 3;
  if (send_items) std::copy(x.send_items.begin(), x.send_items.end(), send_items);
  if (recv_items) std::copy(x.recv_items.begin(), x.recv_items.end(), recv_items);
  *n_send_items = ns;
  *n_recv_items = nr;
  return HDG_OK;
}

// ---- §8(f) NEXT #4: DG-vs-HDG global-matrix size (Tables 1-4 "nonzero ratios"; SPEC.md dg_nnz) ---
hdg_status hdg_nnz_counts(const hdg_mesh* m, const int32_t* dg_ndof, int64_t* nnz_dg, int64_t* nnz_hdg) {
  if (!m || !m->elem_face || !m->face_elem || !m->face_ndof || !dg_ndof || !nnz_dg || !nnz_hdg) return HDG_ERR_ARG;
  const int64_t E = m->n_elem_global, F = m->n_face;
  if (E < 0 || F < 0) return HDG_ERR_ARG;
  for (int64_t i = 0; i < 3 * E; ++i)
    if (m->elem_face[i] < -1 || m->elem_face[i] >= F) return HDG_ERR_ARG;
  for (int64_t f = 0; f < F; ++f) {
    const int32_t l = m->face_elem[2 * f], r = m->face_elem[2 * f + 1];
    if (l < 0 || l >= E || r >= E || m->face_ndof[f] <= 0) return HDG_ERR_ARG;
  }
  // DG (element unknowns coupled through interior faces): one diagonal block per element and one block per
  // neighbour pair in each direction
  int64_t dg = 0;
  for (int64_t e = 0; e < E; ++e) dg += (int64_t)dg_ndof[e] * dg_ndof[e];
  for (int64_t f = 0; f < F; ++f) {
    const int32_t l = m->face_elem[2 * f], r = m->face_elem[2 * f + 1];
    if (r >= 0) dg += 2 * (int64_t)dg_ndof[l] * dg_ndof[r];
  }
  // HDG skeleton (trace unknowns): block row f couples the faces of its one or two elements (diagonal included)
  int64_t hdg = 0;
  for (int64_t f = 0; f < F; ++f) {
    int32_t cols[6];
    int nc = 0;
    for (int side = 0; side < 2; ++side) {
      const int32_t e = m->face_elem[2 * f + side];
      if (e < 0) continue;
      for (int k = 0; k < 3; ++k) {
        const int32_t c = m->elem_face[3 * e + k];
        if (c < 0) continue;
        bool seen = false;
        for (int q = 0; q < nc; ++q) seen |= cols[q] == c;
        if (!seen) cols[nc++] = c;
      }
    }
    for (int q = 0; q < nc; ++q) hdg += (int64_t)m->face_ndof[f] * m->face_ndof[cols[q]];
  }
  *nnz_dg = dg;
  *nnz_hdg = hdg;
  return HDG_OK;
}

// ---- §8(f) NEXT #2: saved local solutions ------------------------------------------------------
static hdg_status solutions_call(hdg_ctx ctx, int mode, const char* name, const void* factors, const double* B,
                                 const double* r_e, const double* X, const double* lambda, double* out,
                                 hdg_stream stream) {
  if (!ctx) return HDG_ERR_ARG;
  const Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "%s: no plan", name);
  ctx->launches = 0;
  if (p.n == 0) return HDG_OK;
  const void* ptrs0[] = {factors, B, r_e, out};
  const void* ptrs1[] = {X, out};
  if (mode == 0) {
    for (const void* q : ptrs0)
      if (!q || !aligned16(q)) return fail(ctx, HDG_ERR_ARG, "%s: null or misaligned (16 B) pointer", name);
  } else {
    for (const void* q : ptrs1)
      if (!q || !aligned16(q)) return fail(ctx, HDG_ERR_ARG, "%s: null or misaligned (16 B) pointer", name);
    if (!lambda && p.n_trace > 0) return fail(ctx, HDG_ERR_ARG, "%s: null lambda", name);
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  for (const Bucket& b : p.buckets) {
    SolutionsArgs a{};
    a.factors = static_cast<const unsigned char*>(factors);
    a.B = B; a.re = r_e; a.lambda = lambda;
    a.X = mode == 0 ? out : nullptr;
    a.Xin = X;
    a.u = mode == 1 ? out : nullptr;
    a.elems = b.d_elems;
    a.offB = p.d_off[OFF_B]; a.offRe = p.d_off[OFF_RE]; a.offF = p.d_off[OFF_F]; a.offX = p.d_off[OFF_X];
    a.offU = p.d_off[OFF_U];
    a.elem_face = p.d_elem_face; a.face_ndof = p.d_face_ndof; a.face_off = p.d_face_off;
    a.elem_begin = p.eb;
    a.ne = b.ne; a.nf = b.nf; a.count = b.count;
    if (mode == 0) HDG_CUDA(ctx, launch_save_solutions(a, ctx->sms, s, &ctx->launches));
    else HDG_CUDA(ctx, launch_backsub_saved(a, ctx->sms, s, &ctx->launches));
  }
  return HDG_OK;
}

hdg_status hdg_save_solutions(hdg_ctx ctx, const void* factors, const double* B, const double* r_e, double* X,
                              hdg_stream stream) {
  return solutions_call(ctx, 0, "hdg_save_solutions", factors, B, r_e, nullptr, nullptr, X, stream);
}

hdg_status hdg_backsubstitute_saved(hdg_ctx ctx, const double* X, const double* lambda, double* u, hdg_stream stream) {
  return solutions_call(ctx, 1, "hdg_backsubstitute_saved", nullptr, nullptr, nullptr, X, lambda, u, stream);
}

// ---- §8(f) NEXT #3: the skeleton solve ----------------------------------------------------
hdg_status hdg_skeleton_spmv(hdg_ctx ctx, const double* K, const double* x, double* y, hdg_stream stream) {
  if (!ctx) return HDG_ERR_ARG;
  const Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "hdg_skeleton_spmv: no plan");
  ctx->launches = 0;
  if (p.sk.f1 == p.sk.f0) return HDG_OK;
  if (!K || !x || !y) return fail(ctx, HDG_ERR_ARG, "hdg_skeleton_spmv: null pointer");
  if (p.max_face_ndof > 32) return fail(ctx, HDG_ERR_UNSUPPORTED, "hdg_skeleton_spmv: face trace size > 32");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  HDG_CUDA(ctx, skeleton_spmv(p, K, x, y, s, &ctx->launches));
  return HDG_OK;
}

hdg_status hdg_skeleton_solve(hdg_ctx ctx, const double* K, const double* E, double* lambda, double rtol, int maxit,
                              int restart, int* iters, double* relres, hdg_stream stream) {
  if (!ctx) return HDG_ERR_ARG;
  Plan& p = ctx->plan;
  if (!p.valid) return fail(ctx, HDG_ERR_STATE, "hdg_skeleton_solve: no plan");
  ctx->launches = 0;
  if (!iters || !relres) return fail(ctx, HDG_ERR_ARG, "hdg_skeleton_solve: null iters/relres");
  if (ctx->nranks != 1 && !ctx->nccl_comm)
    return fail(ctx, HDG_ERR_UNSUPPORTED, "hdg_skeleton_solve: nranks > 1 needs a context with an NCCL communicator");
  if (p.sk.ntr > 0 && (!K || !E || !lambda)) return fail(ctx, HDG_ERR_ARG, "hdg_skeleton_solve: null pointer");
  if (!(rtol > 0.0) || maxit < 1 || restart < 1 || restart > 200)
    return fail(ctx, HDG_ERR_ARG, "hdg_skeleton_solve: rtol > 0, maxit >= 1, 1 <= restart <= 200 required");
  if (p.max_face_ndof > kMaxFaceSolve)
    return fail(ctx, HDG_ERR_UNSUPPORTED, "hdg_skeleton_solve: face trace size %d > %d", p.max_face_ndof, kMaxFaceSolve);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HDG_CUDA(ctx, cudaSetDevice(ctx->device));
  std::string cerr;
  const cudaError_t e = skeleton_gmres(p, p.sw, K, E, lambda, rtol, maxit, restart, s, iters, relres, &ctx->launches,
                                       ctx->nranks > 1 ? ctx->nccl_comm : nullptr, ctx->rank, ctx->nranks, &cerr);
  if (!cerr.empty()) return fail(ctx, HDG_ERR_NCCL, "hdg_skeleton_solve: %s", cerr.c_str());
  if (e == cudaErrorMemoryAllocation) return fail(ctx, HDG_ERR_NOMEM, "hdg_skeleton_solve: workspace");
  if (e != cudaSuccess) return cuda_fail(ctx, e, "hdg_skeleton_solve");
  return HDG_OK;
}

}  // extern "C"



