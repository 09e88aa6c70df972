// nccl_shim.cpp — LD_PRELOAD interposition of NCCL's collective entry points onto libhetccl.so: the
// paper's deployment model, "zero code modification" by "intercepting and overriding NCCL or RCCL
// symbols" (§4.4).
//
//   LD_PRELOAD=paper_2601_22585_b200/libhetccl_nccl.so HETCCL_DOMAINS=0,0,1,1 torchrun ... train.py
//
// * ncclCommInitRank / ncclCommInitRankConfig / ncclCommInitRankScalable: the real NCCL communicator is
//   created first (dlsym RTLD_NEXT); if HETCCL_DOMAINS has one entry per rank (or is unset: one domain),
//   a hetccl communicator for the same ranks is bootstrapped by all-gathering the IPC blobs with the
//   real ncclAllGather, and remembered beside the NCCL one.
// * ncclAllReduce / ncclReduceScatter / ncclAllGather / ncclBroadcast / ncclReduce on such a comm, with
//   a dtype and op hetccl implements (int32 / f16 / f32 / bf16; sum / max / min), run on the hetccl
//   communicator (same stream semantics); anything else goes to the real NCCL unchanged.
// * ncclCommDestroy / ncclCommAbort also destroy the hetccl communicator.
// hetccl_shim_stats() reports how many calls were routed to hetccl and passed through.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/hetccl.h"

namespace {

std::mutex g_mu;
std::unordered_map<ncclComm_t, hetcclComm_t> g_map;
std::atomic<long> g_routed{0}, g_passed{0};

// The real NCCL: RTLD_NEXT finds it when libnccl is in the global scope; Python extension modules load
// it RTLD_LOCAL (torch), so fall back to the already-loaded libnccl.so.2 (RTLD_NOLOAD), else HETCCL_NCCL_LIB.
void* nccl_handle() {
  static void* h = [] {
    void* x = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!x) {
      const char* e = getenv("HETCCL_NCCL_LIB");
      x = dlopen(e && *e ? e : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    }
    return x;
  }();
  return h;
}

template <typename F>
F real(const char* name) {
  static_assert(sizeof(F) == sizeof(void*), "fn ptr");
  void* p = nullptr;
  if (void* h = nccl_handle()) p = dlsym(h, name);
  if (!p) p = dlsym(RTLD_NEXT, name);
  if (!p) {
    fprintf(stderr, "hetccl shim: cannot resolve %s\n", name);
    abort();
  }
  F f;
  memcpy(&f, &p, sizeof(p));
  return f;
}

bool verbose() {
  const char* e = getenv("HETCCL_SHIM_VERBOSE");
  return e && *e && *e != '0';
}

// rank -> domain map for an n-rank communicator, from HETCCL_DOMAINS ("0,0,1,1"); unset: one domain
bool domain_map(int n, std::vector<int>* m) {
  m->assign(n, 0);
  const char* e = getenv("HETCCL_DOMAINS");
  if (!e || !*e) return true;
  std::vector<int> v;
  std::string s(e);
  size_t i = 0;
  while (i <= s.size()) {
    size_t j = s.find(',', i);
    if (j == std::string::npos) j = s.size();
    if (j > i) v.push_back(atoi(s.substr(i, j - i).c_str()));
    i = j + 1;
  }
  if ((int)v.size() != n) return false;
  *m = v;
  return hetccl_validate_map(n, m->data(), nullptr) == hetcclSuccess;
}

// bootstrap a hetccl communicator next to a freshly created NCCL communicator. Every rank takes part in
// both real collectives below whatever happened locally (a rank that skipped them would leave the others
// blocked inside NCCL): the blob all-gather (a rank that failed locally sends an all-zero, invalid blob)
// and an all-reduce(min) of "connected" flags, so either every rank attaches or none does.
void attach(ncclComm_t comm, int nranks, int rank) {
  const char* off = getenv("HETCCL_SHIM_DISABLE");
  if (off && *off && *off != '0') return;
  std::vector<int> m;
  // same decision on every rank: nranks and the environment are shared
  if (nranks < 1 || nranks > HETCCL_MAX_RANKS || !domain_map(nranks, &m)) return;  // (1 rank: the n = 1 copy path)
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t all_bytes = (size_t)nranks * HETCCL_BLOB_BYTES;
  std::vector<char> blob(HETCCL_BLOB_BYTES, 0), all(all_bytes);
  char* d = nullptr;
  if (cudaMalloc((void**)&d, all_bytes + 16) != cudaSuccess) {
    // without a device buffer this rank cannot join the bootstrap collectives: a hang would follow
    fprintf(stderr, "hetccl shim: rank %d cannot allocate the bootstrap buffer; aborting\n", rank);
    abort();
  }
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) st = nullptr;  // legacy stream
  hetcclComm_t hc = nullptr;
  size_t nb = blob.size();
  bool local_ok = hetccl_comm_init(&hc, nranks, rank, m.data(), dev) == hetcclSuccess &&
                  hetccl_comm_export(hc, blob.data(), &nb) == hetcclSuccess;
  if (!local_ok) std::fill(blob.begin(), blob.end(), 0);
  auto ag = real<ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t)>("ncclAllGather");
  auto ar = real<ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t)>(
      "ncclAllReduce");
  bool coll_ok = cudaMemcpy(d + (size_t)rank * HETCCL_BLOB_BYTES, blob.data(), HETCCL_BLOB_BYTES,
                            cudaMemcpyHostToDevice) == cudaSuccess;
  coll_ok = ag(d + (size_t)rank * HETCCL_BLOB_BYTES, d, HETCCL_BLOB_BYTES, ncclInt8, comm, st) == ncclSuccess && coll_ok;
  coll_ok = cudaStreamSynchronize(st) == cudaSuccess && coll_ok;
  coll_ok = cudaMemcpy(all.data(), d, all_bytes, cudaMemcpyDeviceToHost) == cudaSuccess && coll_ok;
  // connect fails (invalid blob) on every rank if any rank failed locally; it can also fail on one rank only
  // (an IPC open), hence the agreement round
  int flag = (local_ok && coll_ok && hetccl_comm_connect(hc, all.data(), all_bytes) == hetcclSuccess) ? 1 : 0;
  int* dflag = (int*)(d + all_bytes);
  bool agreed = cudaMemcpy(dflag, &flag, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess;
  agreed = ar(dflag, dflag, 1, ncclInt32, ncclMin, comm, st) == ncclSuccess && agreed;
  agreed = cudaStreamSynchronize(st) == cudaSuccess && agreed;
  int all_ok = 0;
  agreed = cudaMemcpy(&all_ok, dflag, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess && agreed;
  cudaFree(d);
  if (st) cudaStreamDestroy(st);
  if (!agreed || all_ok != 1) {
    if (verbose()) fprintf(stderr, "hetccl shim: rank %d: bootstrap failed on some rank (local %d), using NCCL\n", rank, flag);
    if (hc) hetccl_comm_destroy(hc);
    return;
  }
  std::lock_guard<std::mutex> l(g_mu);
  g_map[comm] = hc;
  if (verbose()) fprintf(stderr, "hetccl shim: rank %d/%d attached (device %d)\n", rank, nranks, dev);
}

hetcclComm_t lookup(ncclComm_t comm) {
  std::lock_guard<std::mutex> l(g_mu);
  auto it = g_map.find(comm);
  return it == g_map.end() ? nullptr : it->second;
}

// abort = true (ncclCommAbort): forget the hetccl comm without destroying it — destroy synchronises the
// device, which can block for the whole device timeout when a peer is gone; its memory is leaked instead.
void detach(ncclComm_t comm, bool abort_ = false) {
  hetcclComm_t hc = nullptr;
  {
    std::lock_guard<std::mutex> l(g_mu);
    auto it = g_map.find(comm);
    if (it == g_map.end()) return;
    hc = it->second;
    g_map.erase(it);
  }
  if (abort_) {
    if (verbose()) fprintf(stderr, "hetccl shim: abort: hetccl communicator released without device sync\n");
    return;
  }
  hetccl_comm_destroy(hc);
}

bool dt_ok(ncclDataType_t t) { return t == ncclInt32 || t == ncclFloat16 || t == ncclFloat32 || t == ncclBfloat16; }
bool op_ok(ncclRedOp_t o) { return o == ncclSum || o == ncclMax || o == ncclMin; }

ncclResult_t routed(hetcclResult_t r) {
  g_routed++;
  return r == hetcclSuccess ? ncclSuccess : (r == hetcclInvalidArgument ? ncclInvalidArgument : ncclInternalError);
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) void hetccl_shim_stats(long* routed_calls, long* passed_calls) {
  if (routed_calls) *routed_calls = g_routed.load();
  if (passed_calls) *passed_calls = g_passed.load();
}

__attribute__((visibility("default"))) ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id,
                                                                     int rank) {
  ncclResult_t r = real<ncclResult_t (*)(ncclComm_t*, int, ncclUniqueId, int)>("ncclCommInitRank")(comm, nranks, id, rank);
  if (r == ncclSuccess) attach(*comm, nranks, rank);
  return r;
}

__attribute__((visibility("default"))) ncclResult_t ncclCommInitRankConfig(ncclComm_t* comm, int nranks,
                                                                           ncclUniqueId id, int rank,
                                                                           ncclConfig_t* config) {
  ncclResult_t r = real<ncclResult_t (*)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*)>("ncclCommInitRankConfig")(
      comm, nranks, id, rank, config);
  if (r == ncclSuccess && (!config || config->blocking != 0)) attach(*comm, nranks, rank);
  return r;
}

__attribute__((visibility("default"))) ncclResult_t ncclCommInitRankScalable(ncclComm_t* comm, int nranks, int rank,
                                                                             int nId, ncclUniqueId* ids,
                                                                             ncclConfig_t* config) {
  ncclResult_t r = real<ncclResult_t (*)(ncclComm_t*, int, int, int, ncclUniqueId*, ncclConfig_t*)>(
      "ncclCommInitRankScalable")(comm, nranks, rank, nId, ids, config);
  if (r == ncclSuccess && (!config || config->blocking != 0)) attach(*comm, nranks, rank);
  return r;
}

__attribute__((visibility("default"))) ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  detach(comm);
  return real<ncclResult_t (*)(ncclComm_t)>("ncclCommDestroy")(comm);
}

__attribute__((visibility("default"))) ncclResult_t ncclCommAbort(ncclComm_t comm) {
  detach(comm, true);
  return real<ncclResult_t (*)(ncclComm_t)>("ncclCommAbort")(comm);
}

__attribute__((visibility("default"))) ncclResult_t ncclAllReduce(const void* s, void* r, size_t count,
                                                                  ncclDataType_t dt, ncclRedOp_t op, ncclComm_t comm,
                                                                  cudaStream_t st) {
  hetcclComm_t hc = lookup(comm);
  if (hc && dt_ok(dt) && op_ok(op))
    return routed(hetccl_allreduce(s, r, count, (hetcclDataType_t)dt, (hetcclRedOp_t)op, hc, (hetcclStream_t)st));
  g_passed++;
  return real<ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t)>(
      "ncclAllReduce")(s, r, count, dt, op, comm, st);
}

__attribute__((visibility("default"))) ncclResult_t ncclReduceScatter(const void* s, void* r, size_t recvcount,
                                                                      ncclDataType_t dt, ncclRedOp_t op,
                                                                      ncclComm_t comm, cudaStream_t st) {
  hetcclComm_t hc = lookup(comm);
  if (hc && dt_ok(dt) && op_ok(op))
    return routed(hetccl_reduce_scatter(s, r, recvcount, (hetcclDataType_t)dt, (hetcclRedOp_t)op, hc, (hetcclStream_t)st));
  g_passed++;
  return real<ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t)>(
      "ncclReduceScatter")(s, r, recvcount, dt, op, comm, st);
}

__attribute__((visibility("default"))) ncclResult_t ncclAllGather(const void* s, void* r, size_t sendcount,
                                                                  ncclDataType_t dt, ncclComm_t comm, cudaStream_t st) {
  hetcclComm_t hc = lookup(comm);
  if (hc && dt_ok(dt))
    return routed(hetccl_all_gather(s, r, sendcount, (hetcclDataType_t)dt, hc, (hetcclStream_t)st));
  g_passed++;
  return real<ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t)>("ncclAllGather")(
      s, r, sendcount, dt, comm, st);
}

__attribute__((visibility("default"))) ncclResult_t ncclBroadcast(const void* s, void* r, size_t count,
                                                                  ncclDataType_t dt, int root, ncclComm_t comm,
                                                                  cudaStream_t st) {
  hetcclComm_t hc = lookup(comm);
  if (hc && dt_ok(dt))
    return routed(hetccl_broadcast(s, r, count, (hetcclDataType_t)dt, root, hc, (hetcclStream_t)st));
  g_passed++;
  return real<ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t)>(
      "ncclBroadcast")(s, r, count, dt, root, comm, st);
}

__attribute__((visibility("default"))) ncclResult_t ncclReduce(const void* s, void* r, size_t count, ncclDataType_t dt,
                                                               ncclRedOp_t op, int root, ncclComm_t comm,
                                                               cudaStream_t st) {
  hetcclComm_t hc = lookup(comm);
  if (hc && dt_ok(dt) && op_ok(op))
    return routed(hetccl_reduce(s, r, count, (hetcclDataType_t)dt, (hetcclRedOp_t)op, root, hc, (hetcclStream_t)st));
  g_passed++;
  return real<ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t, cudaStream_t)>(
      "ncclReduce")(s, r, count, dt, op, root, comm, st);
}

}  // extern "C"
