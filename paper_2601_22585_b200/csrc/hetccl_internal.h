// hetccl_internal.h — structures shared by the host runtime (plan.cpp, runtime.cu) and the device
// kernels (kernels.cu). Not part of the ABI.
//
// Data layout in HBM:
//   per rank, one cudaMalloc'd, IPC-exported region = [ flags | base | scratch ]
//   flags   : [channel][counter] lines of 128 B; word p of a line counts the signals SENDER p has
//             delivered to this rank on that (channel, counter). Written only by peers
//             (red.release... see kernels.cu), polled locally (ld.acquire.sys), one lane per sender.
//   base    : same shape; this rank's own cumulative "expected so far" per (channel, counter,
//             sender), advanced by each launch at exit, plus the channel's cumulative tile count in
//             word 0 and its cumulative one-shot op count in word 1 of counter line kCounters. Targets are cumulative across launches, so the
//             protocol needs no host sequence numbers and survives CUDA-graph replay.
//   scratch : [channel][slot] ring of nslots (<= kMaxSlots) slots of slot_elems elements; slot g % nslots
//             holds every staging buffer cumulative tile g of that channel needs on this rank.
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace hetccl {

constexpr int kMaxRanks = 16;      // == HETCCL_MAX_RANKS (one flag line = 16 senders x 8 B)
// Two builds of the pipeline kernels (kernels.cu compiled twice):
//   TMA kernels    (namespace k4): 4 CTAs per SM (<= 128 registers), sources staged by TMA bulk copies into a
//                  shared-memory ring — the HBM-bound rank-multiplexed comms;
//   legacy kernels (namespace k2): 2 CTAs per SM (<= 255 registers), sources staged by cp.async — the
//                  NVLink-bound one-rank-per-GPU comms (the round-1 movers measured faster there, r02t/r02y).
constexpr int kCtasPerSm = 4;                      // most resident CTAs per SM of any kernel build
constexpr int kMaxChannels = 148 * kCtasPerSm;     // hard cap on CTAs per rank per op (flag area sizing)
constexpr int kLegacyChannels = 148 * 2;           // default channels of a comm on the legacy kernels
constexpr int kMaxSlots = 16;      // cap on the scratch ring depth per channel (HETCCL_NSLOTS)
#ifndef HETCCL_THREADS
#define HETCCL_THREADS 128
#endif
constexpr int kThreads = HETCCL_THREADS;  // threads per CTA
constexpr int kMaxStages = 5;      // pipeline positions of the deepest op (All-Reduce)
constexpr int kTraceWords = 10;    // per traced iteration: poll start, GO, DONE, fenced, end of stages 0..3;
                                   // iteration 0 also: kernel entry, kernel exit (after the final wait)

// counters (per rank, per channel); C_ACK counts tiles a sender has fully consumed
// C_OS / C_OSACK belong to the one-shot small-message All-Reduce (k_allreduce_oneshot).
enum : int { C_S1 = 0, C_S2 = 1, C_AG = 2, C_S3 = 3, C_ACK = 4, C_OS = 5, C_OSACK = 6, kCounters = 7, C_NONE = 7 };
constexpr size_t kLineWords = 16;  // uint64 words per 128-B line
constexpr size_t kChanWords = (size_t)(kCounters + 1) * kLineWords;  // + one line of channel state
constexpr size_t kFlagsBytes = (size_t)kMaxChannels * kChanWords * sizeof(uint64_t);
constexpr size_t kFlagsReserve = 2 * ((kFlagsBytes + 65535) / 65536) * 65536;  // flags + base, 64K aligned

enum OpKind : int {
  OP_ALLREDUCE = 0,
  OP_REDUCE_SCATTER = 1,
  OP_ALL_GATHER = 2,
  OP_BROADCAST = 3,
  OP_REDUCE = 4,             // NEXT-2: hierarchical Reduce to a root
  OP_ALL_TO_ALL = 5,         // NEXT-2: All-to-All (direct NVLink pushes)
  OP_COPY = 6,
  OP_ALLREDUCE_ONESHOT = 7  // small-message All-Reduce (NEXT-3), same result as OP_ALLREDUCE
};
enum DType : int { DT_INT32 = 2, DT_F16 = 6, DT_F32 = 7, DT_BF16 = 9 };
enum RedOp : int { RED_SUM = 0, RED_MAX = 2, RED_MIN = 3 };

inline int dtype_size(int dt) { return (dt == DT_F16 || dt == DT_BF16) ? 2 : 4; }

// Domain structure, dense ids (reading R4). members[dom_first[k] + j] = j-th rank of
// domain k in ascending order.
struct Topo {
  int n, D, L;  // ranks, domains, lcm of domain sizes
  int dmin;     // smallest domain size
  int rank_dom[kMaxRanks];
  int rank_idx[kMaxRanks];
  int dom_size[kMaxRanks];
  int dom_first[kMaxRanks];
  int members[kMaxRanks];
};

struct RankMem {
  uint64_t* flags;  // as mapped in the launching process/device
  char* scratch;
};

// Per-op, per-rank schedule computed by the host plan (plan.cpp). Pipeline position s of an op is
// the same on every rank; a stage with no work on this rank still holds its position.
//   wait_ctr[s] / wait_mask[s]: before stage s of tile t, every sender in wait_mask must have
//                               signalled counter wait_ctr[s] for tile t;
//   sig_ctr[s]  / sig_mask[s] : after stage s of tile t, signal counter sig_ctr[s] of every rank in
//                               sig_mask (exactly once per tile).
// Consistency (checked by tests): r in sig_mask_w[s] on counter c <=> w in wait_mask_r[s'] where
// wait_ctr_r[s'] == c, with s < s' (a producer always precedes its consumer in the pipeline).
struct RankPlan {
  uint8_t wait_ctr[kMaxStages];
  uint8_t sig_ctr[kMaxStages];
  uint16_t wait_mask[kMaxStages];
  uint16_t sig_mask[kMaxStages];
  uint16_t writes;  // ranks whose scratch this rank writes (ACK wait before reusing a slot)
};

// Kernel parameters (passed by value as a __grid_constant__).
struct OpArgs {
  Topo topo;
  RankMem mem[kMaxRanks];
  RankPlan rp[kMaxRanks];
  const void* send[kMaxRanks];  // per local row (blockIdx.y)
  void* recv[kMaxRanks];
  int local_rank[kMaxRanks];    // rank id of local row
  size_t count;                 // AR/bcast: elements; RS: recvcount; AG: sendcount
  size_t tile;                  // elements per tile (RS/AG: per-shard elements per tile)
  size_t ntiles;
  size_t slot_elems;            // elements per scratch slot
  int nch;
  uint32_t active;              // bitmask of the op's logical stages that are active (same on all ranks)
  int root;
  int op;
  unsigned long long* err;      // device error word of the comm
  long long timeout_ns;
  unsigned long long* trace;    // optional per-iteration timestamps (HETCCL_TRACE_ITERS), else null
  int trace_iters;
  int ws;                       // 0: plain pipeline; k >= 2: warp-specialised, consumers k positions after producers
  int nslots;                   // scratch ring depth (> pipeline positions)
  size_t os_off;                // one-shot area: byte offset in every rank's scratch, bytes per (buffer, sender),
  size_t os_stride;             //   bytes per (buffer, sender, channel) — each channel's region is private to it
  size_t os_chan;
  int final_stage;              // logical stage whose waits become ONE end-of-kernel wait (no pipeline
                                //   position; its work must be empty), or -1
  int direct;                   // 1: every rank's recv buffer is addressable here (peer_recv), so All-Reduce
  void* peer_recv[kMaxRanks];   //    writes final pieces straight into them (no staging through scratch)
  int gpu_scope;                // 1: every rank on this device (rank-multiplexed): flag ops at .gpu scope, else .sys
  int remote_pull;              // 1: pull sources are peers' memory over NVLink (no L2 bulk prefetch of those)
  int flat_ag;                  // 1 (with direct): C writes each final piece into EVERY rank's recv (no stage D)
  int pull;                     // 1 (with direct): every rank's send buffer is addressable (peer_send): the domain
  const void* peer_send[kMaxRanks];  // fold reads peers' x directly, stage A and the s1 staging vanish
  int tma;                      // 1: the movers stage their sources through the TMA ring (dynamic shared memory)
  int l2hint;                   // 1: L2 policies in the TMA movers (evict_first streams, evict_last + discard partials)
  int spacing;                  // plain pipeline (ws == 0): positions between consecutive stages (1 = adjacent)
  int steal;                    // > 0: that percentage of each All-Reduce C stage is published for the rank's other
                                //   channels to take (100: all of it), 0 off
  int steal_help;               // 1: channels that finished their pipeline take published chunks (else owners only)
  int s2g;                      // 1: the TMA movers store results with bulk copies shared -> global
};

// ---- host plan (plan.cpp) ----
int build_topo(int n, const int* map, Topo* t);  // 0 ok, -1 invalid
struct Geometry {
  size_t tile, ntiles;
  int nch;
};
// tile_base: the per-rank All-Reduce tile in bytes (0 = 256 KiB); HETCCL_TILE_KB overrides it
Geometry make_geometry(const Topo& t, int op, size_t count, int es, int nch_max, size_t slot_elems, size_t tile_base);
size_t slot_mult_num(const Topo& t, int op, size_t tile);  // scratch elements one slot needs for `tile`
size_t default_tile_bytes(int op, int n, size_t base);      // HETCCL_TILE_KB or base (AR/BC per rank; RS/AG per shard)
size_t default_slot_bytes(const Topo& t, size_t tile_bytes);  // slot that fits every op's default tile
int op_stages(int op);                                      // logical stages of op
int bcast_relay(const Topo& t, int root);                   // Broadcast: member taking the root's share, or -1
uint32_t active_stages(const Topo& t, int op, int root);   // active logical stages (same on all ranks)
void make_rank_plan(const Topo& t, int op, int rank, int root, RankPlan* rp);
void plan_bytes(const Topo& t, int op, int rank, int root, size_t count, int es, size_t tile, size_t* sent,
                size_t* recv);

// NVLS (nvls.cu, opt-in): multicast-object All-Reduce for single-process multi-GPU communicators
struct NvlsState;
int nvls_eligible_topo(const Topo& t);
int nvls_create(int n, const int* devs, const Topo& t, size_t bytes_per_rank, int nch, NvlsState** out, char* err,
                size_t errlen);
void nvls_destroy(NvlsState* s);
void nvls_buffer(const NvlsState* s, void** p, size_t* bytes);
int nvls_supports(const NvlsState* s, int dt, int red, const void* send, const void* recv);
int nvls_aliases_staging(const NvlsState* s, int dt, const void* p, size_t bytes);
// one rank per process: NVLS state begun at comm init (the domain leader creates the multicast object and a
// socket that hands its file descriptor to the members), finished at connect (handle passing, every member's
// device added, memory bound, peers' cross slots / flags opened through CUDA IPC)
struct NvlsBlob {
  int enabled;         // this rank began NVLS set-up
  char sock[44];       // domain leader: abstract unix-socket name (no leading NUL), else empty
  char ipc[64];        // cudaIpcMemHandle_t of this rank's cross slots + flags
};
int nvls_proc_begin(const Topo& t, int rank, int dev, size_t bytes_per_rank, int nch, NvlsState** out, NvlsBlob* blob,
                    char* err, size_t errlen);
int nvls_proc_connect(NvlsState* s, const Topo& t, int rank, const NvlsBlob* const* blobs, long long timeout_ns,
                      char* err, size_t errlen);

}  // namespace hetccl
