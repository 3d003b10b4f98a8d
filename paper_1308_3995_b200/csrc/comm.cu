// comm.cu — row a7 transport inside libhdg: the NCCL communicator of a context and the
// stream-ordered exchange of shared-face skeleton contributions between element slabs.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2: the copy torch already loaded into the process if any,
// else the system one), so libhdg has no link-time NCCL dependency and single-rank use never touches it.
// The exchange is ONE grouped set of point-to-point calls on the caller's stream:
//     ncclGroupStart; for each peer: ncclRecv(recv slice), ncclSend(send slice); ncclGroupEnd
// between the pack kernel (producer of send) and the ordered accumulate kernel (consumer of recv), all three on
// the same stream — no host synchronization, the accumulate cannot start before the receives have landed, and
// the next step's pack cannot overwrite send before the sends have read it (stream order).
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <vector>

#include <nccl.h>

#include "hdg_internal.cuh"

namespace hdg {
namespace {

struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  std::string err;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      a.h = dlopen(n, RTLD_NOW | RTLD_NOLOAD);   // the copy already in the process (torch's), if any
      if (a.h) break;
    }
    for (const char* n : names) {
      if (a.h) break;
      a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!a.h) {
      a.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return;
    }
#define HDG_SYM(field, name)                                                    \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(a.h, name));            \
  if (!a.field) { a.err = std::string("NCCL symbol missing: ") + name; return; }
    HDG_SYM(getUniqueId, "ncclGetUniqueId");
    HDG_SYM(commInitRank, "ncclCommInitRank");
    HDG_SYM(commDestroy, "ncclCommDestroy");
    HDG_SYM(send, "ncclSend");
    HDG_SYM(recv, "ncclRecv");
    HDG_SYM(groupStart, "ncclGroupStart");
    HDG_SYM(groupEnd, "ncclGroupEnd");
    HDG_SYM(errorString, "ncclGetErrorString");
    HDG_SYM(allReduce, "ncclAllReduce");
    HDG_SYM(broadcast, "ncclBroadcast");
#undef HDG_SYM
  });
  return a;
}

std::string nccl_msg(const char* what, ncclResult_t r) {
  NcclApi& a = api();
  return std::string(what) + ": " + (a.errorString ? a.errorString(r) : "NCCL error");
}

}  // namespace

bool nccl_available(std::string* err) {
  NcclApi& a = api();
  if (a.err.empty()) return true;
  if (err) *err = a.err;
  return false;
}

bool nccl_unique_id(unsigned char* out, std::string* err) {
  if (!nccl_available(err)) return false;
  ncclUniqueId id;
  const ncclResult_t r = api().getUniqueId(&id);
  if (r != ncclSuccess) {
    if (err) *err = nccl_msg("ncclGetUniqueId", r);
    return false;
  }
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return true;
}

bool nccl_comm_init(void** comm, int nranks, int rank, const unsigned char* id_bytes, std::string* err) {
  if (!nccl_available(err)) return false;
  ncclUniqueId id;
  std::memcpy(id.internal, id_bytes, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  const ncclResult_t r = api().commInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) {
    if (err) *err = nccl_msg("ncclCommInitRank", r);
    return false;
  }
  *comm = c;
  return true;
}

void nccl_comm_destroy(void* comm) {
  if (comm && nccl_available(nullptr)) api().commDestroy(static_cast<ncclComm_t>(comm));
}

// One grouped exchange of the packed shared-face contributions (layout of hdg_exchange_counts) on stream s.
bool nccl_exchange(void* comm, const Plan& p, int rank, int nranks, const double* send, double* recv, cudaStream_t s,
                   std::string* err) {
  NcclApi& a = api();
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ncclResult_t r = a.groupStart();
  if (r != ncclSuccess) { if (err) *err = nccl_msg("ncclGroupStart", r); return false; }
  for (int q = 0; q < nranks && r == ncclSuccess; ++q) {
    if (q == rank) continue;
    if (p.sk.recv_counts[q] > 0)
      r = a.recv(recv + p.sk.recv_displs[q], (size_t)p.sk.recv_counts[q], ncclFloat64, q, c, s);
    if (r == ncclSuccess && p.sk.send_counts[q] > 0)
      r = a.send(send + p.sk.send_displs[q], (size_t)p.sk.send_counts[q], ncclFloat64, q, c, s);
  }
  const ncclResult_t r2 = a.groupEnd();
  if (r != ncclSuccess) { if (err) *err = nccl_msg("ncclSend/ncclRecv", r); return false; }
  if (r2 != ncclSuccess) { if (err) *err = nccl_msg("ncclGroupEnd", r2); return false; }
  return true;
}

// sum over ranks, in place, on stream s (the distributed skeleton solve's dot products)
bool nccl_allreduce_sum(void* comm, double* buf, size_t n, cudaStream_t s, std::string* err) {
  const ncclResult_t r = api().allReduce(buf, buf, n, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm), s);
  if (r != ncclSuccess) {
    if (err) *err = nccl_msg("ncclAllReduce", r);
    return false;
  }
  return true;
}

// every rank's segment [off[r], off[r] + cnt[r]) of buf from rank r to all (one group of broadcasts, in place)
bool nccl_allgatherv_inplace(void* comm, int nranks, const std::vector<int64_t>& off, const std::vector<int64_t>& cnt,
                             double* buf, cudaStream_t s, std::string* err) {
  NcclApi& a = api();
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ncclResult_t r = a.groupStart();
  for (int q = 0; q < nranks && r == ncclSuccess; ++q)
    if (cnt[q] > 0) r = a.broadcast(buf + off[q], buf + off[q], (size_t)cnt[q], ncclFloat64, q, c, s);
  const ncclResult_t r2 = a.groupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess) {
    if (err) *err = nccl_msg("ncclBroadcast", r != ncclSuccess ? r : r2);
    return false;
  }
  return true;
}

// grouped point-to-point exchange of per-peer segments: send[peer] (count, offset) from sbuf, recv[peer] into rbuf
bool nccl_p2p(void* comm, int rank, int nranks, const std::vector<int64_t>& scnt, const std::vector<int64_t>& sdsp,
              const double* sbuf, const std::vector<int64_t>& rcnt, const std::vector<int64_t>& rdsp, double* rbuf,
              cudaStream_t s, std::string* err) {
  NcclApi& a = api();
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ncclResult_t r = a.groupStart();
  for (int q = 0; q < nranks && r == ncclSuccess; ++q) {
    if (q == rank) continue;
    if (rcnt[q] > 0) r = a.recv(rbuf + rdsp[q], (size_t)rcnt[q], ncclFloat64, q, c, s);
    if (r == ncclSuccess && scnt[q] > 0) r = a.send(sbuf + sdsp[q], (size_t)scnt[q], ncclFloat64, q, c, s);
  }
  const ncclResult_t r2 = a.groupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess) {
    if (err) *err = nccl_msg("ncclSend/ncclRecv (halo)", r != ncclSuccess ? r : r2);
    return false;
  }
  return true;
}

}  // namespace hdg
