// runtime.cu — host runtime behind include/hetccl.h: communicators (multi-process IPC bootstrap,
// single-process multi-GPU, rank-multiplexed), argument validation and kernel launch. Every
// data-moving step runs in kernels.cu; this file only allocates, maps and enqueues.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unistd.h>
#include <vector>

#include "../../include/hetccl.h"
#include "hetccl_internal.h"

namespace hetccl {
namespace k4 {  // kernels.cu: TMA movers, 4 CTAs per SM
cudaError_t launch_collective(const OpArgs& a, int nlocal, int dt, int red, bool cooperative, cudaStream_t s);
cudaError_t launch_copy(const void* src, void* dst, size_t n, int es, cudaStream_t s);
int max_coresident(int op, int dt, int red, int tma);
}  // namespace k4
namespace k2 {  // kernels_legacy.cu: cp.async movers, 2 CTAs per SM
cudaError_t launch_collective(const OpArgs& a, int nlocal, int dt, int red, bool cooperative, cudaStream_t s);
int max_coresident(int op, int dt, int red, int tma);
}  // namespace k2
cudaError_t nvls_allreduce(NvlsState* s, const void* send, void* recv, size_t count, int dt, unsigned long long* err,
                           long long timeout_ns, cudaStream_t st);
}  // namespace hetccl

using namespace hetccl;

enum CommKind { KIND_PROC = 0, KIND_MUX = 1, KIND_ALL = 2 };

struct hetcclComm {
  int kind = KIND_PROC;
  int n = 0, rank = 0, device = 0;
  int map[kMaxRanks] = {0};
  Topo topo{};
  int nch_max = kMaxChannels;
  size_t tile_base = 0;                   // per-rank All-Reduce tile (0 = 256 KiB; <= 64 channels 1 MiB; mux 4 MiB)
  size_t slot_bytes = 0;
  size_t alloc_bytes = 0;
  char* local[kMaxRanks] = {nullptr};    // allocations owned by this comm (mux: one per rank)
  char* mapped[kMaxRanks] = {nullptr};   // every rank's region as seen from this device
  bool ipc_opened[kMaxRanks] = {false};  // mapped[r] came from cudaIpcOpenMemHandle
  unsigned long long* err = nullptr;     // device error word
  bool connected = false;
  long long timeout_ns = 30LL * 1000000000LL;
  int trace_iters = 0;                    // HETCCL_TRACE_ITERS: per-iteration timestamps of the last op
  int ws = 0;                             // HETCCL_WS: 0 plain pipeline, k in 2..4 warp-specialised (spacing k)
  int direct = 1;                         // HETCCL_DIRECT: write All-Reduce results straight into peers' recv
  int tma = 1;                            // HETCCL_TMA: movers stage sources through the TMA shared-memory ring
  int legacy = 0;                         // HETCCL_LEGACY: pipeline ops on the legacy kernels (k2), else k4
  int nslots = 8;                         // HETCCL_NSLOTS: scratch ring depth
  size_t os_bytes = 0;                    // HETCCL_ONESHOT_KB: one-shot AR up to this many bytes per rank
  size_t os_plain_bytes = 0;              // HETCCL_ONESHOT_PLAIN_KB: the cutoff when recv is not a symmetric buffer
  size_t os_chan = 0;                     // bytes per (buffer, sender, channel): each channel owns its region
  size_t os_stride = 0;                   // bytes per (buffer, sender) of the one-shot area = nch_max * os_chan
  int mid_nch = 128;                      // HETCCL_MID_NCH: channel cap of one-shot and mid-size All-Reduce
  size_t mid_bytes = 0;                   // HETCCL_MID_MB: pipelined All-Reduce up to this size takes the cap
  unsigned long long* trace = nullptr;
  size_t trace_bytes = 0;
  int trace_shape[2] = {0, 0};            // local ranks, channels of the last traced op
  // symmetric buffers (hetccl_mem_*): same size on every rank, peers' copies mapped here
  struct SymBuf {
    char* base = nullptr;
    size_t bytes = 0;
    bool owned = false;                   // allocated by hetccl_mem_alloc
    bool connected = false;
    char* peer[kMaxRanks] = {nullptr};
    bool ipc[kMaxRanks] = {false};
  };
  std::vector<SymBuf> sym;
  NvlsState* nvls = nullptr;              // HETCCL_NVLS=1: per-domain multicast All-Reduce (nvls.cu), else null
  NvlsState* nvls_pending = nullptr;      // one rank per process: begun at init, finished at connect
  NvlsBlob nvls_blob{};
  std::string last_error;
};

namespace {

struct Blob {
  uint32_t magic;
  int version;
  int n, rank;
  int map[kMaxRanks];
  unsigned long long slot_bytes;
  int nch_max;
  int ws;
  int nslots;
  unsigned long long os_bytes;
  unsigned long long os_plain_bytes;
  int mid_nch;
  unsigned long long mid_bytes;
  cudaIpcMemHandle_t handle;
  NvlsBlob nvls;
};
static_assert(sizeof(Blob) <= HETCCL_BLOB_BYTES, "blob too large");
constexpr uint32_t kMagic = 0x48435431u;  // "HCT1"

hetcclResult_t fail(hetcclComm_t c, hetcclResult_t r, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    c->last_error = buf;
  }
  return r;
}

#define CUDA_TRY(c, call)                                                                                  \
  do {                                                                                                     \
    cudaError_t e_ = (call);                                                                               \
    if (e_ != cudaSuccess) return fail((c), hetcclUnhandledCudaError, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

long env_long(const char* name, long dflt) {
  const char* e = getenv(name);
  return e && *e ? atol(e) : dflt;
}

// [flags | base | nch_max x nslots slots | one-shot area: 2 buffers x n senders x nch_max channels x os_chan]
// One-shot regions are private per channel: channel ch's double buffer (parity of ITS op counter) and its
// ACK only order that channel's own reuse, so a region must never be shared between channels of different
// ops (the channel count follows the message size).
constexpr size_t kOsChanMin = 32768;
void set_os_layout(hetcclComm* c) {
  const size_t cut = std::max(c->os_bytes, c->os_plain_bytes);
  const size_t per = (cut + (size_t)c->nch_max - 1) / (size_t)c->nch_max;
  // at least kOsChanMin per channel so mid one-shot sizes can run on fewer, fuller channels (run_op)
  c->os_chan = cut ? (std::max<size_t>(per, kOsChanMin) + 256 + 255) / 256 * 256 : 0;
  c->os_stride = (size_t)c->nch_max * c->os_chan;
}
size_t scratch_slots_bytes(const hetcclComm* c) { return (size_t)c->nch_max * c->nslots * c->slot_bytes; }
size_t alloc_bytes_for(const hetcclComm* c) {
  return kFlagsReserve + scratch_slots_bytes(c) + 2 * (size_t)c->topo.n * c->os_stride;
}

void read_env(hetcclComm* c) {
  // one-rank-per-GPU comms default to the legacy kernels (NVLink-bound; r02y/r02z), rank-multiplexed comms to
  // the TMA kernels (HBM-bound; r02k)
  c->legacy = env_long("HETCCL_LEGACY", c->kind == KIND_MUX ? 0 : 1) != 0;
  c->nch_max = (int)std::max(1L, std::min((long)kMaxChannels,
                                          env_long("HETCCL_NCHANNELS", c->legacy ? kLegacyChannels : kMaxChannels)));
  // small SM budgets (the DDP hook's 64 CTAs): 1 MiB tiles amortise the per-tile protocol (r02bt, r02cb: 256 MiB
  // 348 -> 413 GB/s, 25 MiB buckets 6.2 -> 5.4 ms at 64 CTAs); HETCCL_TILE_KB still overrides
  if (c->kind != KIND_MUX && c->tile_base == 0 && c->nch_max <= 64) c->tile_base = (size_t)1 << 20;
  // scratch slot: HETCCL_SLOT_KB, else sized from this map so every op's default tile fits
  const long slot_kb = env_long("HETCCL_SLOT_KB", 0);
  c->slot_bytes = slot_kb > 0 ? (size_t)std::max(64L, slot_kb) * 1024
                              : default_slot_bytes(c->topo, default_tile_bytes(OP_ALLREDUCE, c->topo.n, c->tile_base));
  c->slot_bytes = (c->slot_bytes + 255) / 256 * 256;
  c->timeout_ns = (long long)std::max(1L, env_long("HETCCL_TIMEOUT_S", 30)) * 1000000000LL;
  c->trace_iters = (int)std::max(0L, std::min(4096L, env_long("HETCCL_TRACE_ITERS", 0)));
  c->ws = (int)env_long("HETCCL_WS", 0);
  c->direct = env_long("HETCCL_DIRECT", 1) != 0;
  c->tma = env_long("HETCCL_TMA", 1) != 0;
  if (c->ws == 1 || c->ws < 0) c->ws = 0;
  if (c->ws > 4) c->ws = 4;
  // rank-multiplexed comms: 6 slots (the deepest op pipeline, staged All-Reduce, has 5 positions) of the larger
  // tile; one-rank-per-GPU comms keep 8
  c->nslots = (int)std::max(2L, std::min((long)kMaxSlots, env_long("HETCCL_NSLOTS", c->kind == KIND_MUX ? 6 : 8)));
  // one-shot cutoff: a rank pushes (n-1) x its buffer, so bound that (16 MiB) rather than the buffer
  // (measured with CUDA graphs: 1+1 one-shot beats the pipeline up to 16 MiB; 2+2 up to ~4 MiB)
  const long os_default_kb = c->topo.n > 1 ? 16384L / (c->topo.n - 1) : 0;
  c->os_bytes = (size_t)std::max(0L, env_long("HETCCL_ONESHOT_KB", os_default_kb)) * 1024;
  // plain (non-symmetric) recv buffers: the pipelined path stages results through scratch, so the one-shot
  // wins up to twice the cutoff (r02ch / r02ci: 1+1 at 24 / 32 MiB 302 / 326 vs 244 / 277 GB/s, 2+2 at 6 MiB
  // 149 vs 124; symmetric buffers lose there). Rank-multiplexed comms always write results directly.
  const long os_plain_default_kb = (long)(c->os_bytes >> 10) * (c->kind == KIND_MUX ? 1 : 2);
  c->os_plain_bytes = (size_t)std::max(0L, env_long("HETCCL_ONESHOT_PLAIN_KB", os_plain_default_kb)) * 1024;
  set_os_layout(c);
  // mid sizes (r02bv/r02bw, 2+2): one tile per channel either way, and 128 channels of larger tiles beat 296 of
  // small ones from 2 to 32 MiB (0.89-1.03x NCCL vs 0.74-0.91x); 1+1 keeps every channel for its pipelined sizes
  // (> 16 MiB: 0.85-0.99x at 128 vs 0.87-1.06x), so the pipelined cap applies only where a domain has >= 2 ranks
  c->mid_nch = (int)std::max(1L, std::min((long)kMaxChannels, env_long("HETCCL_MID_NCH", 128)));
  int dmax = 1;
  for (int k = 0; k < c->topo.D; k++) dmax = std::max(dmax, c->topo.dom_size[k]);
  c->mid_bytes = (size_t)std::max(0L, env_long("HETCCL_MID_MB", dmax >= 2 ? 32 : 0)) << 20;
  c->alloc_bytes = alloc_bytes_for(c);
}

// allocate one rank's [flags | scratch] region on the current device, flags zeroed
cudaError_t alloc_region(size_t bytes, char** out) {
  cudaError_t e = cudaMalloc((void**)out, bytes);
  if (e != cudaSuccess) return e;
  return cudaMemset(*out, 0, kFlagsReserve);
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool valid_dt(int dt) { return dt == DT_INT32 || dt == DT_F16 || dt == DT_F32 || dt == DT_BF16; }
bool valid_red(int op) { return op == RED_SUM || op == RED_MAX || op == RED_MIN; }

bool overlaps(const void* a, size_t an, const void* b, size_t bn) {
  uintptr_t a0 = (uintptr_t)a, b0 = (uintptr_t)b;
  return a0 < b0 + bn && b0 < a0 + an;
}

// NCCL in-place rules; returns nullptr if fine else a message
const char* check_overlap(int op, const void* s, void* r, size_t count, int es, int rank, int n) {
  const size_t b = count * (size_t)es;
  switch (op) {
    case OP_ALLREDUCE:
    case OP_BROADCAST:
      if (s && s != r && overlaps(s, b, r, b)) return "send and recv overlap (only sendbuf == recvbuf is allowed)";
      return nullptr;
    case OP_REDUCE_SCATTER:
      if ((const char*)r == (const char*)s + (size_t)rank * b) return nullptr;
      if (overlaps(s, b * n, r, b)) return "send and recv overlap (in place requires recvbuf == sendbuf + rank*recvcount)";
      return nullptr;
    case OP_ALL_GATHER:
      if ((const char*)s == (const char*)r + (size_t)rank * b) return nullptr;
      if (overlaps(s, b, r, b * n)) return "send and recv overlap (in place requires sendbuf == recvbuf + rank*sendcount)";
      return nullptr;
    case OP_REDUCE:
      if (r && s != r && overlaps(s, b, r, b)) return "send and recv overlap (only sendbuf == recvbuf is allowed)";
      return nullptr;
    case OP_ALL_TO_ALL:
      if (overlaps(s, b * n, r, b * n)) return "all-to-all send and recv must not overlap";
      return nullptr;
  }
  return nullptr;
}

// the elements each rank's recvbuf holds for op (for the n == 1 copy)
size_t recv_elems(int op, size_t count, int n) { return (op == OP_ALL_GATHER || op == OP_ALL_TO_ALL) ? count * n : count; }

hetcclResult_t run_op(hetcclComm_t c, int op, const void* const* sends, void* const* recvs, size_t count, int dt,
                      int red, int root, cudaStream_t stream) {
  if (!c) return hetcclInvalidArgument;
  if (!c->connected) return fail(c, hetcclInvalidUsage, "comm is not connected");
  if (!valid_dt(dt)) return fail(c, hetcclInvalidArgument, "unknown dtype %d", dt);
  if ((op == OP_ALLREDUCE || op == OP_REDUCE_SCATTER || op == OP_REDUCE) && !valid_red(red))
    return fail(c, hetcclInvalidArgument, "unknown reduction op %d", red);
  if ((op == OP_BROADCAST || op == OP_REDUCE) && (root < 0 || root >= c->n))
    return fail(c, hetcclInvalidArgument, "root %d not in [0,%d)", root, c->n);
  const int es = dtype_size(dt);
  if (count > ((size_t)1 << 62) / (size_t)es / (size_t)c->n) return fail(c, hetcclInvalidArgument, "count too large");
  if (count == 0) return hetcclSuccess;
  const int nlocal = c->kind == KIND_MUX ? c->n : 1;
  for (int i = 0; i < nlocal; i++) {
    const int r = c->kind == KIND_MUX ? i : c->rank;
    const bool need_send = !(op == OP_BROADCAST && r != root);
    const bool need_recv = !(op == OP_REDUCE && r != root);
    if ((need_send && !sends[i]) || (need_recv && !recvs[i]))
      return fail(c, hetcclInvalidArgument, "null buffer for rank %d", r);
    const char* msg = check_overlap(op, sends[i], recvs[i], count, es, r, c->n);
    if (msg) return fail(c, hetcclInvalidArgument, "rank %d: %s", r, msg);
  }
  // buffers must be device memory of the comm's device (else hetcclInvalidUsage)
  for (int i = 0; i < nlocal; i++) {
    const void* ps[2] = {sends[i], recvs[i]};
    for (const void* p : ps) {
      if (!p) continue;
      cudaPointerAttributes at;
      if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, hetcclInvalidUsage, "buffer %p is not CUDA memory", p);
      }
      if ((at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) || at.device != c->device)
        return fail(c, hetcclInvalidUsage, "buffer %p is not device memory of the comm's device %d (type %d, device %d)",
                    p, c->device, (int)at.type, at.device);
    }
  }
  DevGuard g(c->device);
  if (c->n == 1) {  // a9: recv <- send
    if (recvs[0]) CUDA_TRY(c, k4::launch_copy(sends[0], recvs[0], recv_elems(op, count, 1), es, stream));
    return hetcclSuccess;
  }
  if (op == OP_ALLREDUCE && c->nvls && nvls_supports(c->nvls, dt, red, sends[0], recvs[0])) {
    if ((((uintptr_t)sends[0] | (uintptr_t)recvs[0]) & 15) != 0)
      return fail(c, hetcclInvalidArgument, "NVLS mode needs 16-byte aligned send/recv buffers");
    if (nvls_aliases_staging(c->nvls, dt, sends[0], count * es) || nvls_aliases_staging(c->nvls, dt, recvs[0], count * es))
      return fail(c, hetcclInvalidArgument,
                  "NVLS buffer is the fp32 staging area of 16-bit All-Reduces (HETCCL_NVLS_WIDE=1): use it for f32 only");
    CUDA_TRY(c, nvls_allreduce(c->nvls, sends[0], recvs[0], count, dt, c->err, c->timeout_ns, stream));
    return hetcclSuccess;
  }
  // symmetric recv (every rank's recv at the same offset of a connected hetccl_mem_* buffer, the direct-mode
  // contract below) takes the one-shot up to os_bytes, a plain recv up to os_plain_bytes
  bool sym_recv = c->kind == KIND_MUX;
  if (op == OP_ALLREDUCE && !sym_recv && c->direct) {
    const char* y = (const char*)recvs[0];
    for (auto& b : c->sym)
      if (b.connected && y >= b.base && y + count * (size_t)es <= b.base + b.bytes) sym_recv = true;
  }
  const size_t os_cut = sym_recv ? c->os_bytes : c->os_plain_bytes;
  bool oneshot = op == OP_ALLREDUCE && os_cut > 0 && count * (size_t)es <= os_cut;
  OpArgs a;
  memset(&a, 0, sizeof(a));
  a.topo = c->topo;
  // rank-multiplexed: every rank runs on this device, so the flag protocol needs only GPU scope
  // (HETCCL_SYS_SCOPE=1 keeps .sys, for A/B)
  a.gpu_scope = c->kind == KIND_MUX && env_long("HETCCL_SYS_SCOPE", 0) != 1;
  for (int r = 0; r < c->n; r++) {
    a.mem[r].flags = (uint64_t*)c->mapped[r];
    a.mem[r].scratch = c->mapped[r] + kFlagsReserve;
    make_rank_plan(c->topo, op, r, root, &a.rp[r]);
  }
  for (int i = 0; i < nlocal; i++) {
    a.send[i] = sends[i];
    a.recv[i] = recvs[i];
    a.local_rank[i] = c->kind == KIND_MUX ? i : c->rank;
  }
  int nch_max = c->nch_max;
  if (c->kind != KIND_MUX) {  // every channel's CTA must be co-resident (the pipeline waits across channels)
    const int cap = (c->legacy && !oneshot) ? k2::max_coresident(op, dt, red, c->tma)
                                            : k4::max_coresident(oneshot ? OP_ALLREDUCE_ONESHOT : op, dt, red, c->tma);
    if (cap > 0) nch_max = std::min(nch_max, cap);
  }
  if (c->kind == KIND_MUX) {
    const int cap = (c->legacy && !oneshot) ? k2::max_coresident(op, dt, red, c->tma)
                                            : k4::max_coresident(oneshot ? OP_ALLREDUCE_ONESHOT : op, dt, red, c->tma);
    if (cap < nlocal) return fail(c, hetcclInternalError, "device cannot co-schedule %d ranks", nlocal);
    nch_max = std::min(nch_max, cap / nlocal);
  }
  const size_t bytes = count * (size_t)es;
  if (oneshot) {  // NEXT-3: one round trip; ~8 KiB of every rank's buffer per channel up to mid_nch channels, then
    // up to kOsChanMin per channel, then every channel (r02bw: 128 channels 1.03-1.74x NCCL at 2-4 MiB vs
    // 0.86-1.57x on 256-296; from 8 MiB the chunk grows past 32 KiB and more channels win again)
    const size_t want = std::max<size_t>(std::min<size_t>((bytes + 8191) / 8192, (size_t)c->mid_nch),
                                         (bytes + kOsChanMin - 1) / kOsChanMin);
    const size_t fit = c->os_chan ? (bytes + c->os_chan - 257) / (c->os_chan - 256) : 1;
    a.nch = (int)std::max<size_t>(1, std::min<size_t>((size_t)nch_max, std::max(want, fit)));
    // the kernel's per-channel chunk (a multiple of the vector width) must fit the channel's private region
    const size_t V = 16 / (size_t)es;
    const size_t chunk = (count + (size_t)a.nch * V - 1) / ((size_t)a.nch * V) * V;
    oneshot = chunk * (size_t)es <= c->os_chan && a.nch <= c->nch_max;
  }
  if (oneshot) {
    a.op = OP_ALLREDUCE_ONESHOT;
    a.count = count;
    a.os_off = scratch_slots_bytes(c);
    a.os_stride = c->os_stride;
    a.os_chan = c->os_chan;
    a.err = c->err;
    a.timeout_ns = c->timeout_ns;
    CUDA_TRY(c, k4::launch_collective(a, nlocal, dt, red, c->kind == KIND_MUX, stream));
    return hetcclSuccess;
  }
  if (c->kind != KIND_MUX && op == OP_ALLREDUCE && bytes <= c->mid_bytes) nch_max = std::min(nch_max, c->mid_nch);
  const size_t slot_elems = c->slot_bytes / (size_t)es;
  Geometry geo = make_geometry(c->topo, op, count, es, nch_max, slot_elems, c->tile_base);
  if (slot_mult_num(c->topo, op, geo.tile) > slot_elems)
    return fail(c, hetcclInternalError, "scratch slot too small for this domain map (raise HETCCL_SLOT_KB)");
  a.count = count;
  a.tile = geo.tile;
  a.ntiles = geo.ntiles;
  a.nch = geo.nch;
  a.slot_elems = slot_elems;
  a.root = root;
  a.op = op;
  a.active = active_stages(c->topo, op, root);
  a.err = c->err;
  a.timeout_ns = c->timeout_ns;
  a.ws = c->ws;
  a.nslots = c->nslots;
  a.tma = c->tma;
  a.spacing = (int)std::max(1L, std::min(4L, env_long("HETCCL_SPACING", 1)));
  // chunk stealing of C stages (opt-in: it evens the channels' finish times, 60-100 us spread instead of 150-270,
  // but the claims cost more than the tail they remove: r02an/r02ao mux 503-505 -> 473-476 GB/s)
  // HETCCL_STEAL = the percentage of each C stage published for stealing (100: all of it), 0 off
  a.steal = op == OP_ALLREDUCE ? (int)std::max(0L, std::min(100L, env_long("HETCCL_STEAL", 0))) : 0;
  a.steal_help = (int)env_long("HETCCL_STEAL_HELP", 1);
  // results leave the TMA movers as bulk copies shared -> global (r02at: mux 501 -> 517 GB/s; across GPUs on the
  // TMA kernels 2+2 at 148 channels 513 -> 530, 1+1 376 -> 446)
  a.s2g = (int)env_long("HETCCL_S2G", 1);
  a.l2hint = (int)env_long("HETCCL_L2HINT", 1);  // evict_first streams (r02n: +4%; partial keep/discard bits 2/4 lose)
  // direct recv mode: in a rank-multiplexed comm every rank's recv buffer is a local pointer; with one
  // rank per GPU, when recvbuf lies in a connected symmetric buffer (hetccl_mem_*), at the same offset in
  // every peer's copy
  a.final_stage = -1;
  if (op == OP_ALLREDUCE && c->kind == KIND_MUX && c->direct) {
    a.direct = 1;
    for (int r = 0; r < c->n; r++) a.peer_recv[r] = recvs[r];
  } else if (op == OP_ALLREDUCE && c->direct) {
    const char* y = (const char*)recvs[0];
    for (auto& b : c->sym)
      if (b.connected && y >= b.base && y + count * (size_t)es <= b.base + b.bytes) {
        a.direct = 1;
        for (int r = 0; r < c->n; r++) a.peer_recv[r] = (r == c->rank ? b.base : b.peer[r]) + (y - b.base);
        break;
      }
  }
  // direct All-Reduce: stage E has no data, only its S3 wait (my y is complete) -> one end-of-kernel wait
  if (a.direct && env_long("HETCCL_FINAL_WAIT", 1)) a.final_stage = 4;
  // flat cross all-gather (direct only): the cross-domain all-gather delivers each final piece to every
  // member of the other domains instead of their segment owner, so the intra-domain forwarding stage D
  // disappears. Same NVLink bytes per rank, more of them cross domains (the paper's hierarchy minimises
  // those): a deviation for NVSwitch (R20). HETCCL_FLAT_AG: 1 always, 0 never, unset = messages of
  // at most HETCCL_FLAT_AG_MAX_KB (32768) per rank, where one tile per channel walks the stages serially
  // and dropping one stage pays (q16, 2+2: 8 MiB +19%, 16 MiB +11%, 32 MiB +4%; 64 MiB and up ±0..2%).
  // With the TMA movers it pays at every size (r02k: 4+4 mux 430 -> 466 GB/s, stage D re-read y from HBM to
  // forward it; r02w: 2+2 / 1+1 at 256 MiB 584 -> 592 / 544 -> 572 GB/s), so the band is unbounded by default.
  // With unequal domains it would load the smallest domain's members (their pieces go to every member of the
  // larger domains: 1+3's singleton sends 2S instead of S), so across GPUs it is on for equal domains only.
  const long flat_env = env_long("HETCCL_FLAT_AG", -1);
  bool equal = true;
  for (int k = 1; k < c->topo.D; k++) equal = equal && c->topo.dom_size[k] == c->topo.dom_size[0];
  const bool flat_band = c->kind == KIND_MUX ||
                         (equal && count * (size_t)es <= (size_t)env_long("HETCCL_FLAT_AG_MAX_KB", 1L << 30) * 1024);
  if (a.direct && a.final_stage == 4 && c->topo.D > 1 && (flat_env == 1 || (flat_env < 0 && flat_band))) {
    a.flat_ag = 1;
    a.active &= ~(1u << 3);
    for (int r = 0; r < c->n; r++) {
      const uint32_t all = ((1u << c->n) - 1u) & ~(1u << r);
      a.rp[r].sig_ctr[2] = C_S3;  // C signals every rank; the end-of-kernel wait collects them
      a.rp[r].sig_mask[2] = (uint16_t)all;
      a.rp[r].wait_ctr[3] = C_NONE;
      a.rp[r].wait_mask[3] = 0;
      a.rp[r].sig_ctr[3] = C_NONE;
      a.rp[r].sig_mask[3] = 0;
      a.rp[r].wait_ctr[4] = C_S3;
      a.rp[r].wait_mask[4] = (uint16_t)all;
      a.rp[r].writes |= (uint16_t)all;
    }
  }
  // pull: every rank's send buffer addressable too (mux, or sendbuf in a symmetric buffer at the same offset
  // on every rank) -> the domain fold reads peers' x directly; stage A and its S1 handshake disappear
  // HETCCL_PULL: 1 always, 0 never, unset = rank-multiplexed comms only (measured: mux +37%; one rank per GPU
  // at 2+2 -10%, because plain 16-byte loads keep too few remote bytes in flight per CTA)
  const long pull_env = env_long("HETCCL_PULL", -1);
  if (a.direct && (pull_env == 1 || (pull_env < 0 && c->kind == KIND_MUX))) {
    if (c->kind == KIND_MUX) {
      a.pull = 1;
      for (int r = 0; r < c->n; r++) a.peer_send[r] = sends[r];
    } else {
      const char* x = (const char*)sends[0];
      for (auto& b : c->sym)
        if (b.connected && x >= b.base && x + count * (size_t)es <= b.base + b.bytes) {
          a.pull = 1;
          for (int r = 0; r < c->n; r++) a.peer_send[r] = (r == c->rank ? b.base : b.peer[r]) + (x - b.base);
          break;
        }
    }
    if (a.pull) {
      a.remote_pull = c->kind != KIND_MUX;
      a.active &= ~1u;  // no stage A
      for (int r = 0; r < c->n; r++) {
        a.rp[r].sig_ctr[0] = C_NONE;
        a.rp[r].sig_mask[0] = 0;
        a.rp[r].wait_ctr[1] = C_NONE;  // readiness is the start round instead
        a.rp[r].wait_mask[1] = 0;
      }
    }
  }
  {  // the ring must be deeper than the pipeline (plus the one-iteration release lag of the WS mode)
    int na = 0;
    for (int s = 0; s < kMaxStages; s++) na += (a.active >> s) & 1;
    const int sp = c->ws >= 2 ? c->ws : std::max(1, a.spacing);
    const int npos = sp * (na - 1) + 1 + (c->ws >= 2 ? 1 : 0);
    if (c->nslots <= npos)
      return fail(c, hetcclInvalidUsage, "HETCCL_NSLOTS=%d must exceed the pipeline depth %d", c->nslots, npos);
  }
  if (c->trace_iters > 0) {
    const size_t need = (size_t)nlocal * geo.nch * c->trace_iters * kTraceWords * sizeof(unsigned long long);
    if (need > c->trace_bytes) {
      if (c->trace) cudaFree(c->trace);
      c->trace = nullptr;
      c->trace_bytes = 0;
      CUDA_TRY(c, cudaMalloc((void**)&c->trace, need));
      c->trace_bytes = need;
    }
    CUDA_TRY(c, cudaMemsetAsync(c->trace, 0, need, stream));
    a.trace = c->trace;
    a.trace_iters = c->trace_iters;
    c->trace_shape[0] = nlocal;
    c->trace_shape[1] = geo.nch;
  }
  if (c->legacy) CUDA_TRY(c, k2::launch_collective(a, nlocal, dt, red, c->kind == KIND_MUX, stream));
  else CUDA_TRY(c, k4::launch_collective(a, nlocal, dt, red, c->kind == KIND_MUX, stream));
  return hetcclSuccess;
}

hetcclResult_t init_common(hetcclComm* c, int n, const int* map) {
  if (build_topo(n, map, &c->topo)) return hetcclInvalidArgument;
  c->n = n;
  memcpy(c->map, map, sizeof(int) * n);
  read_env(c);
  return hetcclSuccess;
}

}  // namespace

extern "C" {

hetcclResult_t hetccl_get_version(int* version) {
  if (!version) return hetcclInvalidArgument;
  *version = HETCCL_VERSION;
  return hetcclSuccess;
}

hetcclResult_t hetccl_validate_map(int nranks, const int* rank_to_domain, int* ndomains) {
  Topo t;
  if (build_topo(nranks, rank_to_domain, &t)) return hetcclInvalidArgument;
  if (ndomains) *ndomains = t.D;
  return hetcclSuccess;
}

hetcclResult_t hetccl_comm_init(hetcclComm_t* comm, int nranks, int rank, const int* rank_to_domain,
                                int cuda_device) {
  if (!comm) return hetcclInvalidArgument;
  *comm = nullptr;
  if (rank < 0 || rank >= nranks) return hetcclInvalidArgument;
  hetcclComm* c = new hetcclComm();
  if (init_common(c, nranks, rank_to_domain) != hetcclSuccess) {
    delete c;
    return hetcclInvalidArgument;
  }
  c->kind = KIND_PROC;
  c->rank = rank;
  c->device = cuda_device;
  DevGuard g(cuda_device);
  cudaError_t e = alloc_region(c->alloc_bytes, &c->local[0]);
  if (e == cudaSuccess) e = cudaMalloc((void**)&c->err, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(c->err, 0, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (c->local[0]) cudaFree(c->local[0]);
    delete c;
    return hetcclUnhandledCudaError;
  }
  c->mapped[rank] = c->local[0];
  if (nranks == 1) c->connected = true;
  // HETCCL_NVLS=1 (opt-in, NEXT-1) with one rank per process: the domain leader creates the multicast object now;
  // connect hands it to the members (hetccl_comm_nvls reports whether the comm ended up in NVLS mode)
  if (nranks > 1 && env_long("HETCCL_NVLS", 0) == 1) {
    char why[256] = {0};
    const size_t mb = (size_t)std::max(1L, env_long("HETCCL_NVLS_MB", 128));
    const int nch = (int)std::max(1L, std::min(1024L, env_long("HETCCL_NVLS_NCH", 148)));
    if (nvls_proc_begin(c->topo, rank, cuda_device, mb << 20, nch, &c->nvls_pending, &c->nvls_blob, why, sizeof(why)))
      c->last_error = why;
  }
  *comm = c;
  return hetcclSuccess;
}

hetcclResult_t hetccl_comm_export(hetcclComm_t c, void* blob, size_t* blob_bytes) {
  if (!c || !blob || !blob_bytes) return hetcclInvalidArgument;
  if (c->kind != KIND_PROC) return fail(c, hetcclInvalidUsage, "export is for one-rank-per-process comms");
  if (*blob_bytes < HETCCL_BLOB_BYTES) return fail(c, hetcclInvalidArgument, "blob buffer < HETCCL_BLOB_BYTES");
  Blob b;
  memset(&b, 0, sizeof(b));
  b.magic = kMagic;
  b.version = HETCCL_VERSION;
  b.n = c->n;
  b.rank = c->rank;
  memcpy(b.map, c->map, sizeof(int) * c->n);
  b.slot_bytes = c->slot_bytes;
  b.nch_max = c->nch_max;
  b.ws = c->ws;
  b.nslots = c->nslots;
  b.os_bytes = c->os_bytes;
  b.os_plain_bytes = c->os_plain_bytes;
  b.mid_nch = c->mid_nch;
  b.mid_bytes = c->mid_bytes;
  b.nvls = c->nvls_blob;
  DevGuard g(c->device);
  CUDA_TRY(c, cudaIpcGetMemHandle(&b.handle, c->local[0]));
  memset(blob, 0, HETCCL_BLOB_BYTES);
  memcpy(blob, &b, sizeof(b));
  *blob_bytes = HETCCL_BLOB_BYTES;
  return hetcclSuccess;
}

hetcclResult_t hetccl_comm_connect(hetcclComm_t c, const void* blobs, size_t blob_bytes) {
  if (!c || !blobs) return hetcclInvalidArgument;
  if (c->kind != KIND_PROC) return fail(c, hetcclInvalidUsage, "connect is for one-rank-per-process comms");
  if (c->connected) return hetcclSuccess;
  if (blob_bytes != (size_t)c->n * HETCCL_BLOB_BYTES)
    return fail(c, hetcclInvalidArgument, "expected %d blobs of %d bytes", c->n, HETCCL_BLOB_BYTES);
  DevGuard g(c->device);
  for (int r = 0; r < c->n; r++) {
    Blob b;
    memcpy(&b, (const char*)blobs + (size_t)r * HETCCL_BLOB_BYTES, sizeof(b));
    if (b.magic != kMagic || b.version != HETCCL_VERSION || b.n != c->n || b.rank != r)
      return fail(c, hetcclInvalidUsage, "blob %d is not a hetccl blob for rank %d of %d", r, r, c->n);
    if (memcmp(b.map, c->map, sizeof(int) * c->n) != 0)
      return fail(c, hetcclInvalidUsage, "rank %d passed a different rank_to_domain map", r);
    if (b.slot_bytes != c->slot_bytes || b.nch_max != c->nch_max || b.ws != c->ws || b.nslots != c->nslots ||
        b.os_bytes != c->os_bytes || b.os_plain_bytes != c->os_plain_bytes || b.mid_nch != c->mid_nch || b.mid_bytes != c->mid_bytes)
      return fail(c, hetcclInvalidUsage, "rank %d has different HETCCL_SLOT_KB/NCHANNELS/WS/NSLOTS/ONESHOT_KB/MID_*", r);
    if (r == c->rank) continue;
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(c, hetcclSystemError, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
    c->mapped[r] = (char*)p;
    c->ipc_opened[r] = true;
  }
  c->connected = true;
  // NVLS (one rank per process): only if every rank began it; then every rank must also finish it, agreed
  // through a status word in each rank's region (1 ok, 2 failed) so no two ranks pick different paths
  bool all_nvls = true;
  const NvlsBlob* nb[kMaxRanks];
  for (int r = 0; r < c->n; r++) {
    nb[r] = &((const Blob*)((const char*)blobs + (size_t)r * HETCCL_BLOB_BYTES))->nvls;
    all_nvls = all_nvls && nb[r]->enabled;
  }
  if (c->nvls_pending && all_nvls) {
    char why[256] = {0};
    const bool ok = nvls_proc_connect(c->nvls_pending, c->topo, c->rank, nb, c->timeout_ns, why, sizeof(why)) == 0;
    if (!ok) c->last_error = why;
    auto status = [&](int r) { return (uint64_t*)(c->mapped[r] + kFlagsReserve / 2) + (size_t)kCounters * kLineWords + 8; };
    const uint64_t mine = ok ? 1 : 2;
    bool agree = cudaMemcpy(status(c->rank), &mine, 8, cudaMemcpyHostToDevice) == cudaSuccess && ok;
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < c->n && agree; r++) {
      uint64_t v = 0;
      while (v == 0) {
        if (cudaMemcpy(&v, status(r), 8, cudaMemcpyDeviceToHost) != cudaSuccess) break;
        if (v == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::nanoseconds(c->timeout_ns)) break;
        if (v == 0) usleep(1000);
      }
      agree = v == 1;
    }
    if (agree) {
      c->nvls = c->nvls_pending;
    } else {
      nvls_destroy(c->nvls_pending);
      if (c->last_error.empty()) c->last_error = "NVLS: a rank could not finish the set-up; staying on the P2P path";
    }
    c->nvls_pending = nullptr;
  } else if (c->nvls_pending) {
    nvls_destroy(c->nvls_pending);
    c->nvls_pending = nullptr;
  }
  return hetcclSuccess;
}

hetcclResult_t hetccl_comm_init_all(hetcclComm_t* comms, int ndev, const int* devlist, const int* rank_to_domain) {
  if (!comms || !devlist || ndev < 1) return hetcclInvalidArgument;
  Topo t;
  if (build_topo(ndev, rank_to_domain, &t)) return hetcclInvalidArgument;
  for (int i = 0; i < ndev; i++)
    for (int j = 0; j < i; j++)
      if (devlist[i] == devlist[j]) return hetcclInvalidArgument;  // one rank per device (use mux otherwise)
  hetcclComm* cs[kMaxRanks] = {nullptr};
  int prev;
  cudaGetDevice(&prev);
  hetcclResult_t res = hetcclSuccess;
  for (int i = 0; i < ndev && res == hetcclSuccess; i++) {
    cs[i] = new hetcclComm();
    init_common(cs[i], ndev, rank_to_domain);
    cs[i]->kind = KIND_ALL;
    cs[i]->rank = i;
    cs[i]->device = devlist[i];
    if (cudaSetDevice(devlist[i]) != cudaSuccess || alloc_region(cs[i]->alloc_bytes, &cs[i]->local[0]) != cudaSuccess ||
        cudaMalloc((void**)&cs[i]->err, 8) != cudaSuccess || cudaMemset(cs[i]->err, 0, 8) != cudaSuccess)
      res = hetcclUnhandledCudaError;
    for (int j = 0; j < ndev && res == hetcclSuccess; j++) {
      if (j == i) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devlist[i], devlist[j]);
      if (!can) res = hetcclSystemError;
      cudaError_t e = cudaDeviceEnablePeerAccess(devlist[j], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) res = hetcclUnhandledCudaError;
    }
    if (cudaDeviceSynchronize() != cudaSuccess) res = hetcclUnhandledCudaError;
  }
  if (res == hetcclSuccess) {
    for (int i = 0; i < ndev; i++) {
      for (int r = 0; r < ndev; r++) cs[i]->mapped[r] = cs[r]->local[0];
      cs[i]->connected = true;
      comms[i] = cs[i];
    }
    // HETCCL_NVLS=1 (opt-in, NEXT-1): All-Reduce through per-domain multicast objects (nvls.cu). If the
    // map or the devices do not allow it the comms stay on the P2P path; hetccl_comm_nvls reports which.
    if (env_long("HETCCL_NVLS", 0) == 1) {
      NvlsState* st[kMaxRanks] = {nullptr};
      char why[256] = {0};
      const size_t mb = (size_t)std::max(1L, env_long("HETCCL_NVLS_MB", 128));
      const int nch = (int)std::max(1L, std::min(1024L, env_long("HETCCL_NVLS_NCH", 148)));
      if (nvls_create(ndev, devlist, t, mb << 20, nch, st, why, sizeof(why)) == 0) {
        for (int i = 0; i < ndev; i++) cs[i]->nvls = st[i];
      } else {
        for (int i = 0; i < ndev; i++) cs[i]->last_error = why;
      }
    }
  } else {
    for (int i = 0; i < ndev; i++)
      if (cs[i]) {
        cudaSetDevice(devlist[i]);
        if (cs[i]->local[0]) cudaFree(cs[i]->local[0]);
        if (cs[i]->err) cudaFree(cs[i]->err);
        delete cs[i];
      }
  }
  cudaSetDevice(prev);
  return res;
}

hetcclResult_t hetccl_comm_init_mux(hetcclComm_t* comm, int nranks, const int* rank_to_domain, int cuda_device) {
  if (!comm) return hetcclInvalidArgument;
  *comm = nullptr;
  hetcclComm* c = new hetcclComm();
  if (init_common(c, nranks, rank_to_domain) != hetcclSuccess) {
    delete c;
    return hetcclInvalidArgument;
  }
  c->kind = KIND_MUX;
  c->device = cuda_device;
  DevGuard g(cuda_device);
  {  // all ranks' CTAs must be co-resident: channels per rank <= SMs x CTAs per SM / nranks (every SM slot
     // unless HETCCL_NCHANNELS caps it)
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
    c->legacy = env_long("HETCCL_LEGACY", 0) != 0;
    const int cps = c->legacy ? 2 : kCtasPerSm;
    c->nch_max = (int)std::max(1L, std::min((long)kMaxChannels, env_long("HETCCL_NCHANNELS", kMaxChannels)));
    c->nch_max = std::max(1, std::min(c->nch_max, sms * cps / nranks));
    // rank-multiplexed comms are HBM-bound and their CTAs share one device: large tiles (4 MiB per rank: one
    // tile per channel up to ~300 MiB messages, so the kernel runs as two bulk phases with the least skew
    // coupling; r02ai: 478 -> 497 GB/s at 4+4 256 MiB), shrunk while the scratch (ranks x channels x slots x
    // slot) would exceed HETCCL_SCRATCH_GB (32)
    c->tile_base = (size_t)4 << 20;
    const int nch = c->nch_max;
    const size_t budget = (size_t)std::max(1L, env_long("HETCCL_SCRATCH_GB", 32)) << 30;
    for (;;) {
      read_env(c);  // re-derive the slot from the tile
      c->nch_max = nch;
      if (c->tile_base <= ((size_t)256 << 10) ||
          (size_t)nranks * (size_t)nch * (size_t)c->nslots * c->slot_bytes <= budget)
        break;
      c->tile_base /= 2;
    }
    set_os_layout(c);
    c->alloc_bytes = alloc_bytes_for(c);
  }
  cudaError_t e = cudaSuccess;
  for (int r = 0; r < nranks && e == cudaSuccess; r++) e = alloc_region(c->alloc_bytes, &c->local[r]);
  if (e == cudaSuccess) e = cudaMalloc((void**)&c->err, 8);
  if (e == cudaSuccess) e = cudaMemset(c->err, 0, 8);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    for (int r = 0; r < nranks; r++)
      if (c->local[r]) cudaFree(c->local[r]);
    if (c->err) cudaFree(c->err);
    delete c;
    return hetcclUnhandledCudaError;
  }
  for (int r = 0; r < nranks; r++) c->mapped[r] = c->local[r];
  c->connected = true;
  *comm = c;
  return hetcclSuccess;
}

hetcclResult_t hetccl_comm_destroy(hetcclComm_t c) {
  if (!c) return hetcclInvalidArgument;
  if (c->nvls) nvls_destroy(c->nvls);
  if (c->nvls_pending) nvls_destroy(c->nvls_pending);
  {
    DevGuard g(c->device);
    cudaDeviceSynchronize();
    for (int r = 0; r < kMaxRanks; r++) {
      if (c->ipc_opened[r]) cudaIpcCloseMemHandle(c->mapped[r]);
      if (c->local[r]) cudaFree(c->local[r]);
    }
    if (c->err) cudaFree(c->err);
    if (c->trace) cudaFree(c->trace);
    for (auto& b : c->sym) {
      for (int r = 0; r < kMaxRanks; r++)
        if (b.ipc[r]) cudaIpcCloseMemHandle(b.peer[r]);
      if (b.owned) cudaFree(b.base);
    }
  }
  delete c;
  return hetcclSuccess;
}

hetcclResult_t hetccl_comm_info(hetcclComm_t c, int* rank, int* nranks, int* domain, int* ndomains, int* domain_rank,
                                int* domain_size) {
  if (!c) return hetcclInvalidArgument;
  if (rank) *rank = c->rank;
  if (nranks) *nranks = c->n;
  if (domain) *domain = c->topo.rank_dom[c->rank];
  if (ndomains) *ndomains = c->topo.D;
  if (domain_rank) *domain_rank = c->topo.rank_idx[c->rank];
  if (domain_size) *domain_size = c->topo.dom_size[c->topo.rank_dom[c->rank]];
  return hetcclSuccess;
}

hetcclResult_t hetccl_comm_nvls(hetcclComm_t c, int* enabled, void** buffer, size_t* bytes) {
  if (!c) return hetcclInvalidArgument;
  if (enabled) *enabled = c->nvls != nullptr;
  nvls_buffer(c->nvls, buffer, bytes);
  return hetcclSuccess;
}

hetcclResult_t hetccl_comm_get_async_error(hetcclComm_t c) {
  if (!c) return hetcclInvalidArgument;
  unsigned long long v = 0;
  DevGuard g(c->device);
  CUDA_TRY(c, cudaMemcpy(&v, c->err, sizeof(v), cudaMemcpyDeviceToHost));
  if (v) return fail(c, hetcclInternalError, "device-side timeout waiting on counter %llu", v >> 8);
  return hetcclSuccess;
}

const char* hetccl_get_error_string(hetcclResult_t r) {
  switch (r) {
    case hetcclSuccess: return "no error";
    case hetcclUnhandledCudaError: return "unhandled cuda error";
    case hetcclSystemError: return "system error (IPC / host)";
    case hetcclInternalError: return "internal error (device timeout or protocol failure)";
    case hetcclInvalidArgument: return "invalid argument";
    case hetcclInvalidUsage: return "invalid usage";
  }
  return "unknown result code";
}

const char* hetccl_get_last_error(hetcclComm_t c) { return c ? c->last_error.c_str() : "null comm"; }

hetcclResult_t hetccl_allreduce(const void* sendbuf, void* recvbuf, size_t count, hetcclDataType_t dt,
                                hetcclRedOp_t op, hetcclComm_t comm, hetcclStream_t stream) {
  if (comm && comm->kind == KIND_MUX) return fail(comm, hetcclInvalidUsage, "use hetccl_mux_* on a mux comm");
  return run_op(comm, OP_ALLREDUCE, &sendbuf, &recvbuf, count, dt, op, 0, (cudaStream_t)stream);
}
hetcclResult_t hetccl_reduce_scatter(const void* sendbuf, void* recvbuf, size_t recvcount, hetcclDataType_t dt,
                                     hetcclRedOp_t op, hetcclComm_t comm, hetcclStream_t stream) {
  if (comm && comm->kind == KIND_MUX) return fail(comm, hetcclInvalidUsage, "use hetccl_mux_* on a mux comm");
  return run_op(comm, OP_REDUCE_SCATTER, &sendbuf, &recvbuf, recvcount, dt, op, 0, (cudaStream_t)stream);
}
hetcclResult_t hetccl_all_gather(const void* sendbuf, void* recvbuf, size_t sendcount, hetcclDataType_t dt,
                                 hetcclComm_t comm, hetcclStream_t stream) {
  if (comm && comm->kind == KIND_MUX) return fail(comm, hetcclInvalidUsage, "use hetccl_mux_* on a mux comm");
  return run_op(comm, OP_ALL_GATHER, &sendbuf, &recvbuf, sendcount, dt, RED_SUM, 0, (cudaStream_t)stream);
}
hetcclResult_t hetccl_reduce(const void* sendbuf, void* recvbuf, size_t count, hetcclDataType_t dt, hetcclRedOp_t op,
                             int root, hetcclComm_t comm, hetcclStream_t stream) {
  if (comm && comm->kind == KIND_MUX) return fail(comm, hetcclInvalidUsage, "use hetccl_mux_* on a mux comm");
  return run_op(comm, OP_REDUCE, &sendbuf, &recvbuf, count, dt, op, root, (cudaStream_t)stream);
}
hetcclResult_t hetccl_all_to_all(const void* sendbuf, void* recvbuf, size_t count, hetcclDataType_t dt,
                                 hetcclComm_t comm, hetcclStream_t stream) {
  if (comm && comm->kind == KIND_MUX) return fail(comm, hetcclInvalidUsage, "use hetccl_mux_* on a mux comm");
  return run_op(comm, OP_ALL_TO_ALL, &sendbuf, &recvbuf, count, dt, RED_SUM, 0, (cudaStream_t)stream);
}
hetcclResult_t hetccl_broadcast(const void* sendbuf, void* recvbuf, size_t count, hetcclDataType_t dt, int root,
                                hetcclComm_t comm, hetcclStream_t stream) {
  if (comm && comm->kind == KIND_MUX) return fail(comm, hetcclInvalidUsage, "use hetccl_mux_* on a mux comm");
  return run_op(comm, OP_BROADCAST, &sendbuf, &recvbuf, count, dt, RED_SUM, root, (cudaStream_t)stream);
}

static hetcclResult_t mux_check(hetcclComm_t c, const void* a, const void* b) {
  if (!c || !a || !b) return hetcclInvalidArgument;
  if (c->kind != KIND_MUX) return fail(c, hetcclInvalidUsage, "hetccl_mux_* needs a comm from hetccl_comm_init_mux");
  return hetcclSuccess;
}
hetcclResult_t hetccl_mux_allreduce(const void* const* s, void* const* r, size_t count, hetcclDataType_t dt,
                                    hetcclRedOp_t op, hetcclComm_t c, hetcclStream_t stream) {
  hetcclResult_t e = mux_check(c, s, r);
  return e ? e : run_op(c, OP_ALLREDUCE, s, r, count, dt, op, 0, (cudaStream_t)stream);
}
hetcclResult_t hetccl_mux_reduce_scatter(const void* const* s, void* const* r, size_t recvcount, hetcclDataType_t dt,
                                         hetcclRedOp_t op, hetcclComm_t c, hetcclStream_t stream) {
  hetcclResult_t e = mux_check(c, s, r);
  return e ? e : run_op(c, OP_REDUCE_SCATTER, s, r, recvcount, dt, op, 0, (cudaStream_t)stream);
}
hetcclResult_t hetccl_mux_all_gather(const void* const* s, void* const* r, size_t sendcount, hetcclDataType_t dt,
                                     hetcclComm_t c, hetcclStream_t stream) {
  hetcclResult_t e = mux_check(c, s, r);
  return e ? e : run_op(c, OP_ALL_GATHER, s, r, sendcount, dt, RED_SUM, 0, (cudaStream_t)stream);
}
hetcclResult_t hetccl_mux_reduce(const void* const* s, void* const* r, size_t count, hetcclDataType_t dt,
                                 hetcclRedOp_t op, int root, hetcclComm_t c, hetcclStream_t stream) {
  if (!c || !s || !r) return hetcclInvalidArgument;
  if (c->kind != KIND_MUX) return fail(c, hetcclInvalidUsage, "hetccl_mux_* needs a comm from hetccl_comm_init_mux");
  return run_op(c, OP_REDUCE, s, r, count, dt, op, root, (cudaStream_t)stream);
}
hetcclResult_t hetccl_mux_all_to_all(const void* const* s, void* const* r, size_t count, hetcclDataType_t dt,
                                     hetcclComm_t c, hetcclStream_t stream) {
  hetcclResult_t e = mux_check(c, s, r);
  return e ? e : run_op(c, OP_ALL_TO_ALL, s, r, count, dt, RED_SUM, 0, (cudaStream_t)stream);
}
hetcclResult_t hetccl_mux_broadcast(const void* const* s, void* const* r, size_t count, hetcclDataType_t dt, int root,
                                    hetcclComm_t c, hetcclStream_t stream) {
  hetcclResult_t e = mux_check(c, s, r);
  return e ? e : run_op(c, OP_BROADCAST, s, r, count, dt, RED_SUM, root, (cudaStream_t)stream);
}

hetcclResult_t hetccl_plan_info(int nranks, const int* rank_to_domain, int rank, int op, size_t count,
                                hetcclDataType_t dt, int root, int nchannels, hetcclPlanInfo_t* info) {
  Topo t;
  if (!info || build_topo(nranks, rank_to_domain, &t) || rank < 0 || rank >= nranks || op < 0 || op > 5 ||
      !valid_dt(dt) || ((op == OP_BROADCAST || op == OP_REDUCE) && (root < 0 || root >= nranks)))
    return hetcclInvalidArgument;
  hetcclComm tmp;
  tmp.topo = t;
  read_env(&tmp);
  const int es = dtype_size(dt);
  int nch = nchannels > 0 ? std::min(nchannels, kMaxChannels) : tmp.nch_max;
  if (nchannels <= 0 && op == OP_ALLREDUCE && count * (size_t)es <= tmp.mid_bytes) nch = std::min(nch, tmp.mid_nch);
  Geometry g = make_geometry(t, op, count, es, nch, tmp.slot_bytes / es, tmp.tile_base);
  memset(info, 0, sizeof(*info));
  plan_bytes(t, op, rank, root, count, es, g.tile, &info->bytes_sent, &info->bytes_recv);
  info->tile_elems = g.tile;
  info->ntiles = g.ntiles;
  info->nchannels = g.nch;
  info->nslots = tmp.nslots;
  return hetcclSuccess;
}

hetcclResult_t hetccl_plan_stages(int nranks, const int* rank_to_domain, int rank, int op, int root,
                                  hetcclStagePlan_t* plan) {
  Topo t;
  if (!plan || build_topo(nranks, rank_to_domain, &t) || rank < 0 || rank >= nranks || op < 0 || op > 5 ||
      ((op == OP_BROADCAST || op == OP_REDUCE) && (root < 0 || root >= nranks)))
    return hetcclInvalidArgument;
  RankPlan rp;
  make_rank_plan(t, op, rank, root, &rp);
  memset(plan, 0, sizeof(*plan));
  plan->nstages = op_stages(op);
  plan->active = active_stages(t, op, root);
  for (int s = 0; s < 8; s++) plan->wait_ctr[s] = plan->sig_ctr[s] = C_NONE;
  for (int s = 0; s < kMaxStages; s++) {
    plan->wait_ctr[s] = rp.wait_ctr[s];
    plan->wait_mask[s] = rp.wait_mask[s];
    plan->sig_ctr[s] = rp.sig_ctr[s];
    plan->sig_mask[s] = rp.sig_mask[s];
  }
  plan->writes = rp.writes;
  return hetcclSuccess;
}

hetcclResult_t hetccl_comm_get_trace(hetcclComm_t c, void* host, size_t bytes, int* shape) {
  if (!c || !shape) return hetcclInvalidArgument;
  shape[0] = c->trace_shape[0];
  shape[1] = c->trace_shape[1];
  shape[2] = c->trace_iters;
  const size_t need = (size_t)shape[0] * shape[1] * shape[2] * kTraceWords * sizeof(unsigned long long);
  if (!c->trace || need == 0) {
    shape[0] = shape[1] = shape[2] = 0;
    return hetcclSuccess;
  }
  if (!host) return hetcclSuccess;  // shape query
  if (!host || bytes < need) return fail(c, hetcclInvalidArgument, "trace buffer needs %zu bytes", need);
  DevGuard g(c->device);
  CUDA_TRY(c, cudaDeviceSynchronize());
  CUDA_TRY(c, cudaMemcpy(host, c->trace, need, cudaMemcpyDeviceToHost));
  return hetcclSuccess;
}

// ------------------------------------------------------------ symmetric buffers (NEXT-4)
namespace {
struct MemBlob {
  uint32_t magic;
  int rank;
  int pid;
  int device;
  unsigned long long bytes;
  unsigned long long raw;  // the pointer in the exporting process (used as is within one process)
  cudaIpcMemHandle_t handle;
};
static_assert(sizeof(MemBlob) <= HETCCL_BLOB_BYTES, "mem blob too large");
constexpr uint32_t kMemMagic = 0x48434d31u;  // "HCM1"

hetcclComm::SymBuf* find_sym(hetcclComm* c, const void* p) {
  for (auto& b : c->sym)
    if (b.base == (const char*)p) return &b;
  return nullptr;
}
}  // namespace

hetcclResult_t hetccl_mem_alloc(hetcclComm_t c, size_t bytes, void** ptr) {
  if (!c || !ptr || bytes == 0) return hetcclInvalidArgument;
  if (c->kind == KIND_MUX) return fail(c, hetcclInvalidUsage, "symmetric buffers are for one-rank-per-GPU comms");
  DevGuard g(c->device);
  hetcclComm::SymBuf b;
  CUDA_TRY(c, cudaMalloc((void**)&b.base, bytes));
  b.bytes = bytes;
  b.owned = true;
  c->sym.push_back(b);
  *ptr = b.base;
  return hetcclSuccess;
}

hetcclResult_t hetccl_mem_export(hetcclComm_t c, void* ptr, void* blob, size_t* blob_bytes) {
  if (!c || !ptr || !blob || !blob_bytes) return hetcclInvalidArgument;
  if (*blob_bytes < HETCCL_BLOB_BYTES) return fail(c, hetcclInvalidArgument, "blob buffer < HETCCL_BLOB_BYTES");
  hetcclComm::SymBuf* b = find_sym(c, ptr);
  if (!b) return fail(c, hetcclInvalidArgument, "not a buffer from hetccl_mem_alloc");
  MemBlob m;
  memset(&m, 0, sizeof(m));
  m.magic = kMemMagic;
  m.rank = c->rank;
  m.pid = (int)getpid();
  m.device = c->device;
  m.bytes = b->bytes;
  m.raw = (unsigned long long)(uintptr_t)b->base;
  DevGuard g(c->device);
  CUDA_TRY(c, cudaIpcGetMemHandle(&m.handle, b->base));
  memset(blob, 0, HETCCL_BLOB_BYTES);
  memcpy(blob, &m, sizeof(m));
  *blob_bytes = HETCCL_BLOB_BYTES;
  return hetcclSuccess;
}

hetcclResult_t hetccl_mem_connect(hetcclComm_t c, void* ptr, const void* blobs, size_t blob_bytes) {
  if (!c || !ptr || !blobs) return hetcclInvalidArgument;
  if (!c->connected) return fail(c, hetcclInvalidUsage, "comm is not connected");
  if (blob_bytes != (size_t)c->n * HETCCL_BLOB_BYTES)
    return fail(c, hetcclInvalidArgument, "expected %d blobs of %d bytes", c->n, HETCCL_BLOB_BYTES);
  hetcclComm::SymBuf* b = find_sym(c, ptr);
  if (!b) return fail(c, hetcclInvalidArgument, "not a buffer from hetccl_mem_alloc");
  DevGuard g(c->device);
  for (int r = 0; r < c->n; r++) {
    MemBlob m;
    memcpy(&m, (const char*)blobs + (size_t)r * HETCCL_BLOB_BYTES, sizeof(m));
    if (m.magic != kMemMagic || m.rank != r) return fail(c, hetcclInvalidUsage, "blob %d is not a hetccl mem blob", r);
    if (m.bytes != b->bytes) return fail(c, hetcclInvalidUsage, "rank %d registered %llu bytes, not %zu", r, m.bytes, b->bytes);
    if (r == c->rank) continue;
    if (m.pid == (int)getpid()) {  // same process (hetccl_comm_init_all): peer access is enabled
      b->peer[r] = (char*)(uintptr_t)m.raw;
    } else {
      void* p = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&p, m.handle, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return fail(c, hetcclSystemError, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
      b->peer[r] = (char*)p;
      b->ipc[r] = true;
    }
  }
  b->connected = true;
  return hetcclSuccess;
}

hetcclResult_t hetccl_mem_free(hetcclComm_t c, void* ptr) {
  if (!c || !ptr) return hetcclInvalidArgument;
  for (size_t i = 0; i < c->sym.size(); i++) {
    auto& b = c->sym[i];
    if (b.base != (char*)ptr) continue;
    DevGuard g(c->device);
    cudaDeviceSynchronize();
    for (int r = 0; r < kMaxRanks; r++)
      if (b.ipc[r]) cudaIpcCloseMemHandle(b.peer[r]);
    if (b.owned) cudaFree(b.base);
    c->sym.erase(c->sym.begin() + i);
    return hetcclSuccess;
  }
  return fail(c, hetcclInvalidArgument, "not a buffer from hetccl_mem_alloc");
}

}  // extern "C"
