// hetccl_internal.h — structures shared by the host runtime (plan.cpp, comm.cu, api.cu) and the
// device kernels (kernels.cu). Not part of the ABI.
//
// Data layout in HBM:
//   per rank, one cudaMalloc'd, IPC-exported region  = [ flags | scratch ]
//   flags   : kMaxChannels x kCounters counters, each on its own 128-B line (kFlagStride words)
//             counters C_S1..C_ACK are written by PEERS (red.release.sys.add) and polled locally
//             (ld.acquire.sys); line C_BASE holds this rank's own cumulative "expected" values, so
//             the protocol survives CUDA-graph replay (no host-side sequence numbers).
//   scratch : kMaxChannels x kNumSlots slots of slot_elems elements; a slot holds every staging
//             buffer one tile of one op needs on this rank (layout per op in kernels.cu).
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace hetccl {

constexpr int kMaxRanks = 16;     // == HETCCL_MAX_RANKS
constexpr int kMaxChannels = 64;  // hard cap on CTAs per rank per op
constexpr int kNumSlots = 2;      // scratch ring depth per channel
constexpr int kThreads = 512;     // threads per CTA
constexpr int kFlagStride = 16;   // uint64 words per counter line (128 B)

// counters (per rank, per channel)
enum : int { C_S1 = 0, C_S2 = 1, C_AG = 2, C_S3 = 3, C_ACK = 4, C_NREMOTE = 5, C_BASE = 5, kCounters = 6 };
constexpr size_t kChanWords = (size_t)kCounters * kFlagStride;
constexpr size_t kFlagsBytes = (size_t)kMaxChannels * kChanWords * sizeof(uint64_t);  // 48 KiB
constexpr size_t kFlagsReserve = 64 * 1024;  // scratch starts here (256-B aligned)

enum OpKind : int { OP_ALLREDUCE = 0, OP_REDUCE_SCATTER = 1, OP_ALL_GATHER = 2, OP_BROADCAST = 3, OP_COPY = 4 };
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

// Per-op, per-rank protocol constants computed by the host plan.
struct RankPlan {
  uint32_t partners;      // bitmask of ranks this rank exchanges data with (symmetric)
  uint32_t inc[C_NREMOTE];  // arrivals per tile on each counter (C_ACK: acks per tile)
};

// Kernel parameters (passed by value as a __grid_constant__; < 4 KiB).
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
  int root;
  int op;
  unsigned long long* err;      // device error word of the comm
  long long timeout_ns;
};

// ---- host plan (plan.cpp) ----
int build_topo(int n, const int* map, Topo* t);  // 0 ok, -1 invalid
struct Geometry {
  size_t tile, ntiles;
  int nch;
};
// q = alignment quantum of a tile in elements
Geometry make_geometry(const Topo& t, int op, size_t count, int es, int nch_max, size_t slot_elems);
size_t slot_mult_num(const Topo& t, int op, size_t tile);  // scratch elements one slot needs for `tile`
void make_rank_plan(const Topo& t, int op, int rank, int root, RankPlan* rp);
void plan_bytes(const Topo& t, int op, int rank, int root, size_t count, int es, size_t tile, size_t* sent,
                size_t* recv);

}  // namespace hetccl
