// kernels.cu — sm_100a device code of the hierarchical collectives.
//
// One persistent CTA per (channel, local rank), 128 threads; compiled twice (hetccl_internal.h): the TMA build
// (namespace k4, 4 CTAs per SM, sources staged by TMA bulk copies into a shared-memory ring and results stored by
// bulk copies, "tma_move") and the legacy build (k2, kernels_legacy.cu, 2 CTAs per SM, sources staged by
// cp.async, 16-byte register stores). Every op is a short list
// of stages (All-Reduce: A intra push, B domain fold of the other domains' pieces + cross push, C
// domain fold of my pieces + cross fold + all-gather writes, D intra forward, E completion); a channel
// runs them as a SOFTWARE PIPELINE over its tiles t = ch, ch+nch, ...: iteration i runs the stage at
// position p on the channel's tile i-p, so the intra- and cross-domain stages of different tiles overlap
// and no flag round trip sits on the critical path (run_pipeline). Data moves through the movers below;
// stores go straight into a peer's
// IPC-mapped scratch slot, or — when every rank's recv buffer is addressable (rank-multiplexed comms,
// symmetric buffers) — straight into the peers' recv buffers ("direct"), and the domain fold may read
// the peers' send buffers ("pull", rank-multiplexed comms). Hand-off between stages uses per-(receiver,
// channel, counter, SENDER) counters:
//   writer: data stores -> __syncthreads -> fence.acq_rel.sys -> red.relaxed.sys.add(+1) on the
//           receiver's counter word of this sender;
//   reader: lane p of warp 0 spins ld.acquire.sys on sender p's word until it reaches the
//           cumulative target -> __syncthreads -> loads of the data
// (.gpu instead of .sys when all ranks share this device: rank-multiplexed comms).
// Scratch is a ring of nslots slots per channel indexed by the channel's cumulative tile count;
// before writing a tile's slot a rank waits for the ACK of the tile that last used it. Targets are
// cumulative across launches (kept in the rank's own base lines), so the protocol needs no host
// sequence numbers and replays under CUDA graphs. The same kernels serve the rank-multiplexed mode
// (all ranks on one device, rank = blockIdx.y, cooperative launch) and the one-rank-per-GPU mode.
// Small All-Reduces take k_allreduce_oneshot (one push round, local domain-major reduction).
//
// Arithmetic (readings R3, R5, R6, R8): per element, fold ascending rank inside a domain
// (seeded with the first operand), narrow 16-bit types once at the domain boundary, fold the D
// partials in ascending domain id, narrow once more. fp32 accumulation for bf16/fp16, IEEE RNE
// everywhere (__fadd_rn, __float2bfloat16_rn, __float2half_rn), uint32 wrap for int32. Built
// without --use_fast_math (no FTZ, reading R9).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>

#include "hetccl_internal.h"

// This file is compiled twice (hetccl_internal.h): as is -> namespace hetccl::k4 (TMA movers, 4 CTAs per SM),
// and through kernels_legacy.cu -> namespace hetccl::k2 (cp.async movers, 2 CTAs per SM, no TMA ring).
#ifndef HETCCL_KNS
#define HETCCL_KNS k4
#endif
#ifndef HETCCL_KERNEL_CPS
#define HETCCL_KERNEL_CPS 4
#endif
#ifndef HETCCL_LEGACY_MOVERS
#define HETCCL_LEGACY_MOVERS 0
#endif

namespace hetccl {
namespace HETCCL_KNS {

// ------------------------------------------------------------------ PTX primitives -------------
// Flag operations at system scope (peers are other GPUs, over NVLink) or — when every rank of the
// communicator runs on this device (rank-multiplexed comms, OpArgs::gpu_scope) — at GPU scope, where the
// release fence only has to order this SM's stores at L2 instead of across the fabric.
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p, int gpu) {
  uint64_t v;
  if (gpu) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel(int gpu) {
  if (gpu) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  else asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ void red_add_relaxed(uint64_t* p, uint64_t v, int gpu) {
  if (gpu) asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint32_t ld_s32(const void* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint16_t ld_s16(const void* p) {
  uint16_t v;
  asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_s32(void* p, uint32_t v) {
  asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_s16(void* p, uint16_t v) {
  asm volatile("st.global.u16 [%0], %1;" ::"l"(p), "h"(v) : "memory");
}

// ------------------------------------------------------------------ element traits -------------
template <typename T>
struct Tr;
template <>
struct Tr<float> {
  using S = uint32_t;  // storage word
  using A = float;     // accumulator
  static constexpr int V = 4;
  __device__ static A widen(S s) { return __uint_as_float(s); }
  __device__ static S narrow(A a) { return __float_as_uint(a); }
};
template <>
struct Tr<int32_t> {
  using S = uint32_t;
  using A = uint32_t;  // wraps mod 2^32 (reading R8)
  static constexpr int V = 4;
  __device__ static A widen(S s) { return s; }
  __device__ static S narrow(A a) { return a; }
};
template <>
struct Tr<__nv_bfloat16> {
  using S = uint16_t;
  using A = float;
  static constexpr int V = 8;
  __device__ static A widen(S s) { return __uint_as_float((uint32_t)s << 16); }  // exact
  __device__ static S narrow(A a) { return __bfloat16_as_ushort(__float2bfloat16_rn(a)); }  // RNE
};
template <>
struct Tr<__half> {
  using S = uint16_t;
  using A = float;
  static constexpr int V = 8;
  __device__ static A widen(S s) { return __half2float(__ushort_as_half(s)); }  // exact
  __device__ static S narrow(A a) { return __half_as_ushort(__float2half_rn(a)); }  // RNE, keeps subnormals
};

template <int OP>
__device__ __forceinline__ float comb(float a, float b) {
  if (OP == RED_SUM) return __fadd_rn(a, b);
  if (OP == RED_MAX) return fmaxf(a, b);
  return fminf(a, b);
}
template <int OP>
__device__ __forceinline__ uint32_t comb(uint32_t a, uint32_t b) {
  if (OP == RED_SUM) return a + b;
  if (OP == RED_MAX) return (int32_t)a > (int32_t)b ? a : b;
  return (int32_t)a < (int32_t)b ? a : b;
}

// unpack / pack a 16-byte vector of storage words
template <typename S>
struct Vec;
template <>
struct Vec<uint32_t> {
  __device__ static uint32_t get(const uint4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }
  __device__ static void set(uint4& v, int e, uint32_t s) {
    if (e == 0) v.x = s;
    else if (e == 1) v.y = s;
    else if (e == 2) v.z = s;
    else v.w = s;
  }
};
template <>
struct Vec<uint16_t> {
  __device__ static uint16_t get(const uint4& v, int e) {
    uint32_t w = Vec<uint32_t>::get(v, e >> 1);
    return (uint16_t)((e & 1) ? (w >> 16) : (w & 0xffffu));
  }
  __device__ static void set(uint4& v, int e, uint16_t s) {
    uint32_t w = Vec<uint32_t>::get(v, e >> 1);
    w = (e & 1) ? ((w & 0xffffu) | ((uint32_t)s << 16)) : ((w & 0xffff0000u) | s);
    Vec<uint32_t>::set(v, e >> 1, w);
  }
};

// ------------------------------------------------------------------ CTA data movers ------------
constexpr int kMaxList = kMaxRanks + 2;
struct PtrList {
  const void* p[kMaxList];
  int n;
  uint32_t keep;  // L2 hints (HETCCL_L2HINT): destinations -> store evict_last (read back soon: the cross
                  // partials); sources -> dead after this read (discard their L2 lines, no write-back)
  __device__ PtrList() : n(0), keep(0) {}
  __device__ void add(const void* q) { p[n++] = q; }
  __device__ void add_keep(const void* q) { keep |= 1u << n; p[n++] = q; }
};

__device__ __forceinline__ bool all_aligned16(const PtrList& a, const PtrList& b) {
  uintptr_t o = 0;
  for (int i = 0; i < a.n; i++) o |= (uintptr_t)a.p[i];
  for (int i = 0; i < b.n; i++) o |= (uintptr_t)b.p[i];
  return (o & 15) == 0;
}

// data-thread geometry of the current CTA (set by run_pipeline: warp-specialised CTAs leave warp 0
// to the flag protocol), read by the data movers
__shared__ int g_dbase, g_dnth;
__shared__ int g_pf;  // 1: the movers may L2-prefetch their sources (all local); 0 when folds read peers' memory

#ifndef HETCCL_FOLD_UNROLL
#define HETCCL_FOLD_UNROLL 4
#endif
#ifndef HETCCL_COPY_UNROLL
#define HETCCL_COPY_UNROLL 8
#endif
constexpr int kUnroll = HETCCL_FOLD_UNROLL;      // vectors in flight per thread per source in a fold
constexpr int kCopyUnroll = HETCCL_COPY_UNROLL;  // vectors in flight per thread in a copy

#ifndef HETCCL_PREFETCH
#define HETCCL_PREFETCH 2
#endif
// L2 prefetch, `HETCCL_PREFETCH` batches ahead, of the vectors a CTA-wide batch will load: one TMA bulk
// prefetch per source issued by the first data thread (no registers, no shared memory). Hides the HBM
// latency the register-bound loads cannot (128 threads x 4-8 vectors in flight per CTA).
__device__ __forceinline__ void prefetch_ahead(const void* src, size_t v0, int tid, size_t batch_vecs, size_t nv) {
  if (HETCCL_PREFETCH <= 0 || tid != 0 || !g_pf) return;  // (a bulk prefetch of peer memory stalls ~20x)
  const size_t vs = v0 + (size_t)HETCCL_PREFETCH * batch_vecs;
  if (vs >= nv) return;
  const size_t bytes = min(batch_vecs, nv - vs) * 16;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((const char*)src + vs * 16), "r"((uint32_t)bytes)
               : "memory");
}

#ifndef HETCCL_TMA
#define HETCCL_TMA 1
#endif

// Fold sources are staged through shared memory with cp.async (LDGSTS): each data thread issues the
// 16-byte loads of up to kStageSrc sources x kUnroll vectors at once and waits once, so a fold keeps
// kStageSrc times the bytes in flight that register loads (one source at a time) could, without the
// registers. Each thread reads back only the slots it filled itself (no CTA barrier).
constexpr int kStageSrc = 5;
constexpr int kStageVecs = kStageSrc * kUnroll;  // 16-byte slots per data thread
// the staging slots live in the dynamic shared memory of the legacy (2 CTAs per SM) kernels
extern __shared__ __align__(128) unsigned char g_ring[];
#define g_stage ((uint4*)g_ring)
constexpr size_t kStageBytes = (size_t)kStageVecs * kThreads * 16;
__shared__ int g_lgsts;  // 1: the movers stage through g_stage (legacy kernels), 0: TMA ring or register loads
__device__ __forceinline__ void cp_async16(uint4* sdst, const void* gsrc) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------ TMA-staged movers ----------
// The pipeline kernels' data movers stream their sources through a ring of kTmaStages shared-memory
// stages filled by TMA bulk copies (cp.async.bulk global->shared; completion counted on the stage's FULL
// mbarrier): the first data thread keeps kTmaStages-1 chunks of every operand in flight while every data
// warp folds the oldest chunk out of shared memory and stores the result (16-byte st.global, to every
// destination), then arrives on the stage's EMPTY mbarrier; the producer refills a stage once every data
// warp has arrived. No CTA-wide barrier per chunk: a warp only waits for its data, the producer only for
// the slowest warp of the chunk NST-1 behind. Loads cost no registers or issue slots of the folding
// threads, so the bytes in flight per CTA (~3 x 24 KiB) do not depend on the register budget (the
// LDG/LDGSTS movers of round 1 kept 12% of warps active at 254 registers, profiles/r01/q28). Operand and
// destination pointers live in shared memory for the duration of a call (the PtrLists are on the stack,
// and their local-memory reads missed L1 once the ring took the shared-memory carve-out: r02e).
//   chunk g of this CTA (g counts every chunk of every mover call since kernel start, g_seq) uses stage
//   g % kTmaStages; it is that stage's u-th use (u = g / kTmaStages): FULL phase parity u & 1, and before
//   issuing it the producer waits for EMPTY completion u-1 (parity (u-1) & 1).
#ifndef HETCCL_TMA_STAGES
#define HETCCL_TMA_STAGES 2
#endif
#ifndef HETCCL_TMA_STAGE_KB
#define HETCCL_TMA_STAGE_KB 24  // 2 x 24 KiB per CTA, 4 CTAs per SM: fewer, larger chunks beat deeper rings
#endif                          // (r02ab/r02ac mux: 2x24 478-480, 2x26 475, 3x18 472, 3x16 456, 3x36 @3 CTAs 459)
constexpr int kTmaStages = HETCCL_TMA_STAGES;
constexpr int kTmaStageBytes = HETCCL_TMA_STAGE_KB * 1024;
constexpr int kTmaMaxVpt = 4;  // 16-byte vectors per thread per operand per chunk (register bound of the fold)
#ifndef HETCCL_TMA_ALIGN_V
#define HETCCL_TMA_ALIGN_V 8
#endif
constexpr uint32_t kTmaAlignV = HETCCL_TMA_ALIGN_V;  // chunk granularity in 16-byte vectors
__shared__ __align__(8) uint64_t g_full[kTmaStages];
__shared__ __align__(8) uint64_t g_empty[kTmaStages];
__shared__ unsigned g_seq;  // chunks this CTA has issued/consumed so far (all data threads agree)
__shared__ int g_tma;       // 1: the ring is initialised and the op may use it
__shared__ const char* g_ops[kMaxList + kMaxRanks];  // operands of the current call, in load order
__shared__ char* g_dst[kMaxList];                     // destinations of the current call

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(smem_addr(b)), "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_addr(b))
               : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_addr(b)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_v4_hint(void* p, const uint4& v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_addr(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* gdst, const void* ssrc, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_addr(ssrc)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__shared__ int g_l2hint;  // OpArgs::l2hint of the running op
__shared__ int g_s2g;     // 1: the ring movers store results by TMA bulk copies shared -> global (OpArgs::s2g)
__shared__ uint32_t g_keep_dst, g_dead_ops;  // the current call's hint masks (destinations / operands)
__device__ __forceinline__ void data_bar() { asm volatile("bar.sync 1, %0;" ::"r"(g_dnth) : "memory"); }

// thread 0 at the start of a pipeline kernel, before its first __syncthreads (data warps: all warps, or
// all but the sync warp in the warp-specialised mode)
__device__ __forceinline__ void tma_init(int enable, int data_warps, int l2hint, int s2g) {
  if (threadIdx.x == 0) {
    g_tma = HETCCL_TMA && !HETCCL_LEGACY_MOVERS && enable;
    g_s2g = s2g;
    g_lgsts = HETCCL_LEGACY_MOVERS;
    g_l2hint = l2hint;
    g_seq = 0;
    if (g_tma) {
      for (int s = 0; s < kTmaStages; s++) {
        mbar_init(&g_full[s], 1);
        mbar_init(&g_empty[s], (uint32_t)data_warps);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
}

// operands the ring can stage (at least one warp's vectors of each per chunk), nv vectors in 32 bits
__device__ __forceinline__ bool tma_fits(int nops, size_t nv) {
  return g_tma && nops >= 1 && nops <= kMaxList + kMaxRanks && nops * 16 * (int)max(32u, kTmaAlignV) <= kTmaStageBytes &&
         nv < (1u << 31);
}

// Chunk loop of the movers: operands g_ops[0..nops), destinations g_dst[0..nd) (shared memory), nv
// 16-byte vectors. Kept free of stack state (scalar arguments, 32-bit counters, pointers from shared
// memory): with the ring holding most of the shared-memory carve-out the L1 left for local memory is
// small, and one spilled loop variable reloaded from L2 per chunk cost ~a quarter of the kernel (r02g).
template <typename T, int OP, int MODE>
__device__ __noinline__ void tma_stream(int ni, int D, int kpos, int nd, uint32_t nv, unsigned seq0) {
  using TR = Tr<T>;
  using S = typename TR::S;
  using A = typename TR::A;
  constexpr int V = TR::V;
  const int tid = (int)threadIdx.x - g_dbase, nth = g_dnth;
  const int nops = MODE == 2 ? ni + D - 1 : (MODE == 1 ? ni : 1);
  // vectors per operand per chunk: as many as the stage holds, in whole 128-byte lines (HETCCL_TMA_ALIGN_V
  // vectors) so every bulk copy starts line-aligned in global memory when the operand does
  const uint32_t cv = min((uint32_t)(kTmaStageBytes / (nops * 16)) / kTmaAlignV * kTmaAlignV, (uint32_t)(kTmaMaxVpt * nth));
  const uint32_t chb = cv * 16;
  const uint32_t nchunks = (nv + cv - 1) / cv;
  // L2 policy (HETCCL_L2HINT): every operand and result is touched once, so loads and stores stream with
  // evict_first; the cross partials (keep-masked destinations) are stored evict_last so they are still in L2
  // when their owner's next stage reads them, and after that read (dead-masked operands) their lines are
  // discarded — never written back to HBM.
  // HETCCL_L2HINT bits: 1 evict_first on streamed loads/stores, 2 evict_last on kept stores, 4 discard dead operands
  const int hint = g_l2hint & 3;
  const uint32_t keep = (g_l2hint & 2) ? g_keep_dst : 0u, dead = (g_l2hint & 4) ? g_dead_ops : 0u;
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
  // S2G (HETCCL_S2G): each result vector goes back into operand 0's slot of the stage, and one thread stores the
  // chunk to every destination with bulk copies — one instruction per destination instead of one 16-byte store
  // per thread and vector, which is what limits a CTA pushing to NVLink peers (tools/tma_probe.cu: one TMA
  // thread per CTA pushes ~43 GB/s, r02v)
  const int s2g = g_s2g;
  auto issue = [&](uint32_t cn) {
    const unsigned g = seq0 + cn, st = g % kTmaStages, u = g / kTmaStages;
    if (u > 0) mbar_wait(&g_empty[st], (u - 1) & 1u);  // every data warp is done with the stage's last use
    if (s2g && u > 0) bulk_wait_read();                 // ... and my bulk stores have read it
    const uint32_t bytes = min(cv, nv - cn * cv) * 16;
    mbar_arrive_expect_tx(&g_full[st], bytes * (uint32_t)nops);
    for (int j = 0; j < nops; j++) {
      if (hint & 1) bulk_g2s_hint(g_ring + st * kTmaStageBytes + j * chb, g_ops[j] + (size_t)cn * chb, bytes, &g_full[st], pol_first);
      else bulk_g2s(g_ring + st * kTmaStageBytes + j * chb, g_ops[j] + (size_t)cn * chb, bytes, &g_full[st]);
    }
  };
  if (tid == 0)
    for (uint32_t c = 0; c < nchunks && c < (uint32_t)kTmaStages - 1; c++) issue(c);
  const int lane = threadIdx.x & 31;
  for (uint32_t c = 0; c < nchunks; c++) {
    if (tid == 0 && c + kTmaStages - 1 < nchunks) issue(c + kTmaStages - 1);
    const unsigned g = seq0 + c, st = g % kTmaStages;
    mbar_wait(&g_full[st], (g / kTmaStages) & 1u);
    if (dead) {  // the chunk of every dead operand is in shared memory: drop its whole 128-byte lines from L2
      const uint32_t bytes = min(cv, nv - c * cv) * 16;
      for (int j = 0; j < nops; j++) {
        if (!((dead >> j) & 1u)) continue;
        const uintptr_t a0 = (uintptr_t)(g_ops[j] + (size_t)c * chb), a1 = a0 + bytes;
        for (uintptr_t l = (a0 + 127) / 128 * 128 + (uintptr_t)tid * 128; l + 128 <= a1; l += (uintptr_t)nth * 128)
          discard_l2((const void*)l);
      }
    }
    const unsigned char* sb = g_ring + st * kTmaStageBytes;
    const uint32_t lim = min(cv, nv - c * cv);
    for (uint32_t idx = tid; idx < lim; idx += nth) {
      uint4 o = *(const uint4*)(sb + idx * 16);
      if (MODE != 0) {
        // first operand peeled (no loop-carried "first?" select: it pushed acc[] to local memory, r02j)
        A acc[V];
#pragma unroll
        for (int e = 0; e < V; e++) acc[e] = TR::widen(Vec<S>::get(o, e));
#pragma unroll 1
        for (int j = 1; j < ni; j++) {
          const uint4 w = *(const uint4*)(sb + j * chb + idx * 16);
#pragma unroll
          for (int e = 0; e < V; e++) acc[e] = comb<OP>(acc[e], TR::widen(Vec<S>::get(w, e)));
        }
        if (MODE == 2) {
          uint4 pk;
#pragma unroll
          for (int e = 0; e < V; e++) Vec<S>::set(pk, e, TR::narrow(acc[e]));
          const uint4 w0 = kpos == 0 ? pk : *(const uint4*)(sb + ni * chb + idx * 16);
#pragma unroll
          for (int e = 0; e < V; e++) acc[e] = TR::widen(Vec<S>::get(w0, e));
#pragma unroll 1
          for (int q = 1; q < D; q++) {
            const uint4 w = q == kpos ? pk : *(const uint4*)(sb + (ni + (q < kpos ? q : q - 1)) * chb + idx * 16);
#pragma unroll
            for (int e = 0; e < V; e++) acc[e] = comb<OP>(acc[e], TR::widen(Vec<S>::get(w, e)));
          }
        }
#pragma unroll
        for (int e = 0; e < V; e++) Vec<S>::set(o, e, TR::narrow(acc[e]));
      }
      const size_t off = ((size_t)c * cv + idx) * 16;
      if (s2g) {
        *(uint4*)(sb + idx * 16) = o;  // operand 0's slot: only this thread read it
      } else if (hint == 3) {
        for (int d = 0; d < nd; d++) st_v4_hint(g_dst[d] + off, o, ((keep >> d) & 1u) ? pol_last : pol_first);
      } else if (hint == 2) {
        for (int d = 0; d < nd; d++) {
          if ((keep >> d) & 1u) st_v4_hint(g_dst[d] + off, o, pol_last);
          else st_v4(g_dst[d] + off, o);
        }
      } else if (hint == 1) {
        for (int d = 0; d < nd; d++) st_v4_hint(g_dst[d] + off, o, pol_first);
      } else {
        for (int d = 0; d < nd; d++) st_v4(g_dst[d] + off, o);
      }
    }
    if (s2g) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // my smem results -> the bulk copy engine
      data_bar();
      if (tid == 0) {
        for (int d = 0; d < nd; d++) {
          if (hint & 1) bulk_s2g_hint(g_dst[d] + (size_t)c * chb, sb, lim * 16, ((keep >> d) & 1u) ? pol_last : pol_first);
          else bulk_s2g(g_dst[d] + (size_t)c * chb, sb, lim * 16);
        }
        bulk_commit();
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&g_empty[st]);  // this warp is done with stage st
  }
  if (s2g && tid == 0) bulk_wait_all();  // the stores are complete (visible) before the pipeline's release fence
  *(volatile unsigned*)&g_seq = seq0 + nchunks;  // every data thread writes the same value
}

// ---- chunk stealing inside the ring (HETCCL_STEAL; the C stage of All-Reduce) ----------------------------
// A job is one mover call's chunks, published in a 64-bit word W = tag(16) << 48 | total(24) << 24 | count(24)
// (tag = tile index << 4 | slot of the owning channel; flags line kCounters, word 0, of (rank, channel); word 1
// counts the chunks other channels completed). The owner and any helper claim kClaimBatch chunks at a time with
// one atomicAdd on W, issued a batch AHEAD by the producer thread so the claim's latency hides behind the
// chunks in flight; the claimed index rides to the consumers in g_chunk_of[stage], and an exhausted claim sends
// a sentinel stage (plain arrive, no bytes) that ends the call. An add that lands on an exhausted word is
// harmless (count only grows past total); jobs are only published when every channel has one tile, so a word
// never changes job while a helper holds its tag.
constexpr uint32_t kClaimBatch = 4;
__shared__ uint64_t* g_claim;    // job word of the current dynamic call, or null
__shared__ int g_claim_mode;     // 0 static chunks, 1 owner (publishes W), 2 helper
__shared__ uint64_t g_claim_tag; // the tag the call's operand lists were built for
__shared__ unsigned g_claimed;   // chunks this CTA processed in its last dynamic call
__shared__ unsigned g_job_total; // chunks of the job the owner published (0: none)
__shared__ int g_vec_only;       // 1: the fold movers run only their TMA vector part (helpers; no scalar tail)
__shared__ int g_chunk_of[kTmaStages];
__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t fetch_add_acq_rel(uint64_t* p, uint64_t v) {
  uint64_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
constexpr uint64_t kTagMask = ~((1ull << 48) - 1);

template <typename T, int OP, int MODE>
__device__ __noinline__ void tma_stream_dyn(int ni, int D, int kpos, int nd, uint32_t nv, unsigned seq0) {
  using TR = Tr<T>;
  using S = typename TR::S;
  using A = typename TR::A;
  constexpr int V = TR::V;
  const int tid = (int)threadIdx.x - g_dbase, nth = g_dnth;
  const int nops = MODE == 2 ? ni + D - 1 : (MODE == 1 ? ni : 1);
  const uint32_t cv = min((uint32_t)(kTmaStageBytes / (nops * 16)) / kTmaAlignV * kTmaAlignV, (uint32_t)(kTmaMaxVpt * nth));
  const uint32_t chb = cv * 16;
  const uint32_t nchunks = (nv + cv - 1) / cv;
  const int mode = g_claim_mode;
  uint64_t* w = g_claim;
  const uint64_t tag = g_claim_tag;
  const int hint = g_l2hint & 1;
  const uint64_t pol_first = policy_evict_first();
  if (mode == 1 && tid == 0) {
    *(volatile uint64_t*)(w + 1) = 0;
    g_job_total = nchunks;
    st_release_gpu(w, tag | ((uint64_t)nchunks << 24));  // count 0
  }
  // (producer) claims: the batch being used and the one claimed ahead of it
  bool ended = false;                  // the sentinel is issued
  uint64_t ahead = 0;                  // W before the add that claimed the next batch
  uint32_t cur = 0, cur_end = 0;       // chunks [cur, cur_end) of the current batch are left
  auto claim_batch = [&]() -> uint64_t { return fetch_add_acq_rel(w, kClaimBatch); };
  auto next_chunk = [&]() -> long long {
    if (cur >= cur_end) {  // take the batch claimed ahead, claim the next one
      const uint64_t tot = (ahead >> 24) & 0xffffffull, cnt = ahead & 0xffffffull;
      if ((ahead & kTagMask) != tag || cnt >= tot) return -1;
      cur = (uint32_t)cnt;
      cur_end = (uint32_t)min(tot, cnt + kClaimBatch);
      ahead = claim_batch();
    }
    return cur++;
  };
  const int s2g = g_s2g;
  auto issue = [&](uint32_t k) {
    const unsigned g = seq0 + k, st = g % kTmaStages, u = g / kTmaStages;
    if (u > 0) mbar_wait(&g_empty[st], (u - 1) & 1u);
    if (s2g && u > 0) bulk_wait_read();
    const long long c = next_chunk();
    *(volatile int*)&g_chunk_of[st] = (int)c;
    if (c < 0) {
      ended = true;
      mbar_arrive(&g_full[st]);  // sentinel: completes the phase with no bytes
      return;
    }
    const uint32_t bytes = min(cv, nv - (uint32_t)c * cv) * 16;
    mbar_arrive_expect_tx(&g_full[st], bytes * (uint32_t)nops);
    for (int j = 0; j < nops; j++) {
      if (hint) bulk_g2s_hint(g_ring + st * kTmaStageBytes + j * chb, g_ops[j] + (size_t)c * chb, bytes, &g_full[st], pol_first);
      else bulk_g2s(g_ring + st * kTmaStageBytes + j * chb, g_ops[j] + (size_t)c * chb, bytes, &g_full[st]);
    }
  };
  if (tid == 0) ahead = claim_batch();
  if (tid == 0)
    for (uint32_t k = 0; k < (uint32_t)kTmaStages - 1 && !ended; k++) issue(k);
  const int lane = threadIdx.x & 31;
  uint32_t k = 0, mine = 0;
  for (;;) {
    if (tid == 0 && !ended) issue(k + kTmaStages - 1);
    const unsigned g = seq0 + k, st = g % kTmaStages;
    mbar_wait(&g_full[st], (g / kTmaStages) & 1u);
    const int c = *(volatile int*)&g_chunk_of[st];
    k++;
    if (c < 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&g_empty[st]);
      break;
    }
    unsigned char* sb = g_ring + st * kTmaStageBytes;
    const uint32_t lim = min(cv, nv - (uint32_t)c * cv);
    for (uint32_t idx = tid; idx < lim; idx += nth) {
      uint4 o = *(const uint4*)(sb + idx * 16);
      if (MODE != 0) {
        A acc[V];
#pragma unroll
        for (int e = 0; e < V; e++) acc[e] = TR::widen(Vec<S>::get(o, e));
#pragma unroll 1
        for (int j = 1; j < ni; j++) {
          const uint4 wv = *(const uint4*)(sb + j * chb + idx * 16);
#pragma unroll
          for (int e = 0; e < V; e++) acc[e] = comb<OP>(acc[e], TR::widen(Vec<S>::get(wv, e)));
        }
        if (MODE == 2) {
          uint4 pk;
#pragma unroll
          for (int e = 0; e < V; e++) Vec<S>::set(pk, e, TR::narrow(acc[e]));
          const uint4 w0 = kpos == 0 ? pk : *(const uint4*)(sb + ni * chb + idx * 16);
#pragma unroll
          for (int e = 0; e < V; e++) acc[e] = TR::widen(Vec<S>::get(w0, e));
#pragma unroll 1
          for (int q = 1; q < D; q++) {
            const uint4 wv = q == kpos ? pk : *(const uint4*)(sb + (ni + (q < kpos ? q : q - 1)) * chb + idx * 16);
#pragma unroll
            for (int e = 0; e < V; e++) acc[e] = comb<OP>(acc[e], TR::widen(Vec<S>::get(wv, e)));
          }
        }
#pragma unroll
        for (int e = 0; e < V; e++) Vec<S>::set(o, e, TR::narrow(acc[e]));
      }
      const size_t off = ((size_t)c * cv + idx) * 16;
      if (s2g) {
        *(uint4*)(sb + idx * 16) = o;  // operand 0's slot: only this thread read it
      } else if (hint) {
        for (int d = 0; d < nd; d++) st_v4_hint(g_dst[d] + off, o, pol_first);
      } else {
        for (int d = 0; d < nd; d++) st_v4(g_dst[d] + off, o);
      }
    }
    if (s2g) {  // as in tma_stream: one bulk store per destination
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      data_bar();
      if (tid == 0) {
        for (int d = 0; d < nd; d++) {
          if (hint) bulk_s2g_hint(g_dst[d] + (size_t)c * chb, sb, lim * 16, pol_first);
          else bulk_s2g(g_dst[d] + (size_t)c * chb, sb, lim * 16);
        }
        bulk_commit();
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&g_empty[st]);
    mine++;
  }
  if (s2g && tid == 0) bulk_wait_all();
  *(volatile unsigned*)&g_seq = seq0 + k;  // every data thread writes the same values
  *(volatile unsigned*)&g_claimed = mine;
}

// Vector part (nv 16-byte vectors) of the three movers through the ring:
//   MODE 0 copy : dst[d] = inner[0] (bits)
//   MODE 1 fold : dst[d] = narrow(fold_{s} widen(inner[s]))
//   MODE 2 hier : P = narrow(fold_s widen(inner[s])); dst[d] = narrow(fold_{q < outer.n} widen(q == kpos ? P : outer[q]))
// Operands are staged in load order inner[0..ni), then outer[q] for q != kpos ascending.
template <typename T, int OP, int MODE>
__device__ __forceinline__ void tma_move(const PtrList& inner, int kpos, const PtrList& outer, const PtrList& dsts,
                                         size_t nv) {
  const int tid = (int)threadIdx.x - g_dbase;
  const int ni = inner.n, D = outer.n, nd = dsts.n;
  const int nops = MODE == 2 ? ni + D - 1 : (MODE == 1 ? ni : 1);
  data_bar();  // every data thread is done with the previous call's pointers and has published g_seq
  const unsigned seq0 = *(volatile unsigned*)&g_seq;  // read before the 2nd barrier: no thread can move it on yet
  if (tid < nops) g_ops[tid] = (const char*)(tid < ni ? inner.p[tid] : outer.p[tid - ni < kpos ? tid - ni : tid - ni + 1]);
  if (tid < nd) g_dst[tid] = (char*)dsts.p[tid];
  if (tid == 0) {
    g_keep_dst = dsts.keep;
    // dead operands in load order: inner bits as is, outer bits (q != kpos) after them
    uint32_t dm = inner.keep;
    if (MODE == 2)
      for (int q = 0; q < D; q++)
        if (q != kpos && ((outer.keep >> q) & 1u)) dm |= 1u << (ni + (q < kpos ? q : q - 1));
    g_dead_ops = dm;
  }
  data_bar();
  if (MODE == 2 && g_claim_mode) tma_stream_dyn<T, OP, MODE>(ni, D, kpos, nd, (uint32_t)nv, seq0);
  else tma_stream<T, OP, MODE>(ni, D, kpos, nd, (uint32_t)nv, seq0);
}

// dst[d][i] = src[i] for every destination d, i < n elements of size ES (bit copy)
template <int ES>
__device__ __noinline__ void cta_copy(const void* src, const PtrList& dsts, size_t n) {
  if (n == 0) return;
  constexpr int V = 16 / ES;
  const int tid = (int)threadIdx.x - g_dbase, nth = g_dnth;
  PtrList s1;
  s1.add(src);
  const size_t nv = all_aligned16(s1, dsts) ? n / V : 0;
  const char* sp = (const char*)src;
  size_t nvr = nv;  // vectors left to the register path
  if (nv && tma_fits(1, nv)) {
    PtrList none;
    tma_move<float, RED_SUM, 0>(s1, -1, none, dsts, nv);
    nvr = 0;
  }
  for (size_t v0 = tid; v0 < nvr; v0 += (size_t)kCopyUnroll * nth) {
    prefetch_ahead(sp, v0, tid, (size_t)kCopyUnroll * nth, nv);
    uint4 w[kCopyUnroll];
#pragma unroll
    for (int u = 0; u < kCopyUnroll; u++) {
      size_t v = v0 + (size_t)u * nth;
      if (v < nv) w[u] = ld_v4(sp + v * 16);
    }
    for (int d = 0; d < dsts.n; d++) {
      char* dp = (char*)dsts.p[d];
#pragma unroll
      for (int u = 0; u < kCopyUnroll; u++) {
        size_t v = v0 + (size_t)u * nth;
        if (v < nv) st_v4(dp + v * 16, w[u]);
      }
    }
  }
  for (size_t i = nv * V + tid; i < n; i += nth) {
    if (ES == 4) {
      uint32_t w = ld_s32(sp + i * 4);
      for (int d = 0; d < dsts.n; d++) st_s32((char*)dsts.p[d] + i * 4, w);
    } else {
      uint16_t w = ld_s16(sp + i * 2);
      for (int d = 0; d < dsts.n; d++) st_s16((char*)dsts.p[d] + i * 2, w);
    }
  }
}

template <int ES>
__device__ __forceinline__ void cta_copy1(const void* src, void* dst, size_t n) {
  PtrList d;
  d.add(dst);
  cta_copy<ES>(src, d, n);
}

// dst[d][i] = narrow( fold_{s in order} widen(src[s][i]) ) for every destination d
template <typename T, int OP>
__device__ __noinline__ void cta_fold(const PtrList& srcs, const PtrList& dsts, size_t n) {
  using TR = Tr<T>;
  using S = typename TR::S;
  using A = typename TR::A;
  constexpr int V = TR::V;
  if (n == 0) return;
  if (srcs.n == 1) {  // a single operand: the value is already in the dtype (bit copy)
    cta_copy<sizeof(S)>(srcs.p[0], dsts, n);
    return;
  }
  const int tid = (int)threadIdx.x - g_dbase, nth = g_dnth;
  const size_t nv = all_aligned16(srcs, dsts) ? n / V : 0;
  size_t nvr = nv;  // vectors left to the register path
  if (nv && tma_fits(srcs.n, nv)) {
    PtrList none;
    tma_move<T, OP, 1>(srcs, -1, none, dsts, nv);
    nvr = 0;
  }
  if (g_lgsts) {  // round-1 movers: cp.async staging of the fold sources (legacy kernels)
  for (size_t v0 = tid; v0 < nvr; v0 += (size_t)kUnroll * nth) {
    for (int s = 0; s < srcs.n; s++) prefetch_ahead(srcs.p[s], v0, tid, (size_t)kUnroll * nth, nv);
    A acc[kUnroll][V];
    for (int s0 = 0; s0 < srcs.n; s0 += kStageSrc) {
      const int g = min(kStageSrc, srcs.n - s0);
      for (int j = 0; j < g; j++) {
        const char* sp = (const char*)srcs.p[s0 + j];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
          const size_t v = v0 + (size_t)u * nth;
          if (v < nv) cp_async16(&g_stage[(j * kUnroll + u) * nth + tid], sp + v * 16);
        }
      }
      cp_async_wait_all();
      for (int j = 0; j < g; j++) {
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
          const uint4 w = g_stage[(j * kUnroll + u) * nth + tid];
#pragma unroll
          for (int e = 0; e < V; e++) {
            const A x = TR::widen(Vec<S>::get(w, e));
            acc[u][e] = s0 + j == 0 ? x : comb<OP>(acc[u][e], x);
          }
        }
      }
    }
    uint4 o[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int e = 0; e < V; e++) Vec<S>::set(o[u], e, TR::narrow(acc[u][e]));
    for (int d = 0; d < dsts.n; d++) {
      char* dp = (char*)dsts.p[d];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        size_t v = v0 + (size_t)u * nth;
        if (v < nv) st_v4(dp + v * 16, o[u]);
      }
    }
  }
  } else {
  for (size_t v0 = tid; v0 < nvr; v0 += (size_t)kUnroll * nth) {
    for (int s = 0; s < srcs.n; s++) prefetch_ahead(srcs.p[s], v0, tid, (size_t)kUnroll * nth, nv);
    A acc[kUnroll][V];
    {
      uint4 w[kUnroll];
      const char* sp = (const char*)srcs.p[0];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        size_t v = v0 + (size_t)u * nth;
        if (v < nv) w[u] = ld_v4(sp + v * 16);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; u++)
#pragma unroll
        for (int e = 0; e < V; e++) acc[u][e] = TR::widen(Vec<S>::get(w[u], e));
    }
    for (int s = 1; s < srcs.n; s++) {
      uint4 w[kUnroll];
      const char* sp = (const char*)srcs.p[s];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        size_t v = v0 + (size_t)u * nth;
        if (v < nv) w[u] = ld_v4(sp + v * 16);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; u++)
#pragma unroll
        for (int e = 0; e < V; e++) acc[u][e] = comb<OP>(acc[u][e], TR::widen(Vec<S>::get(w[u], e)));
    }
    uint4 o[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int e = 0; e < V; e++) Vec<S>::set(o[u], e, TR::narrow(acc[u][e]));
    for (int d = 0; d < dsts.n; d++) {
      char* dp = (char*)dsts.p[d];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        size_t v = v0 + (size_t)u * nth;
        if (v < nv) st_v4(dp + v * 16, o[u]);
      }
    }
  }
  }
  for (size_t i = nv * V + tid; i < n; i += nth) {
    A a;
    if (sizeof(S) == 4) a = TR::widen((S)ld_s32((const char*)srcs.p[0] + i * 4));
    else a = TR::widen((S)ld_s16((const char*)srcs.p[0] + i * 2));
    for (int s = 1; s < srcs.n; s++) {
      S w = sizeof(S) == 4 ? (S)ld_s32((const char*)srcs.p[s] + i * 4) : (S)ld_s16((const char*)srcs.p[s] + i * 2);
      a = comb<OP>(a, TR::widen(w));
    }
    S r = TR::narrow(a);
    for (int d = 0; d < dsts.n; d++) {
      if (sizeof(S) == 4) st_s32((char*)dsts.p[d] + i * 4, (uint32_t)r);
      else st_s16((char*)dsts.p[d] + i * 2, (uint16_t)r);
    }
  }
}

// Two-level fold (the hierarchy of reading R3/R6 in one pass):
//   P_kpos = narrow( fold_{s in order} widen(inner[s][i]) ), P_q = outer[q][i] for q != kpos,
//   dst[d][i] = narrow( fold_{q < outer.n in order} widen(P_q) ) for every destination d.
// Used where a rank owns both its domain's partial and the cross-domain result of an element, so the
// partial never round-trips through memory. Bitwise identical to cta_fold of inner, stored, then
// cta_fold of outer.
template <typename T, int OP>
__device__ __noinline__ void cta_fold_hier(const PtrList& inner, int kpos, const PtrList& outer, const PtrList& dsts,
                                           size_t n) {
  using TR = Tr<T>;
  using S = typename TR::S;
  using A = typename TR::A;
  constexpr int V = TR::V;
  if (n == 0) return;
  const int tid = (int)threadIdx.x - g_dbase, nth = g_dnth;
  const int D = outer.n;
  uintptr_t al = 0;
  for (int q = 0; q < D; q++)
    if (q != kpos) al |= (uintptr_t)outer.p[q];
  const size_t nv = (all_aligned16(inner, dsts) && (al & 15) == 0) ? n / V : 0;
  size_t nvr = nv;  // vectors left to the register path
  if (nv && tma_fits(inner.n + D - 1, nv)) {
    tma_move<T, OP, 2>(inner, kpos, outer, dsts, nv);
    nvr = 0;
  }
  if (g_vec_only) return;  // a stealing helper: the owner does everything the ring does not
  if (g_lgsts) {  // round-1 movers: cp.async staging of the fold sources (legacy kernels)
  // operand list in load order: inner[0..inner.n), then outer[q] for q != kpos ascending; staged in groups
  // of kStageSrc (at 4+4 all five operands of a tile batch are in flight at once)
  const int L = inner.n + D - 1;
  auto operand = [&](int j) -> const char* {
    if (j < inner.n) return (const char*)inner.p[j];
    const int q = j - inner.n;
    return (const char*)outer.p[q < kpos ? q : q + 1];
  };
  for (size_t v0 = tid; v0 < nvr; v0 += (size_t)kUnroll * nth) {
    for (int s = 0; s < inner.n; s++) prefetch_ahead(inner.p[s], v0, tid, (size_t)kUnroll * nth, nv);
    for (int q = 0; q < D; q++)
      if (q != kpos) prefetch_ahead(outer.p[q], v0, tid, (size_t)kUnroll * nth, nv);
    int lo = 0, hi = 0;  // operands [lo, hi) are in the staging slots [0, hi - lo)
    auto stage = [&](int j) -> int {
      if (j >= hi) {
        lo = j;
        hi = min(L, j + kStageSrc);
        for (int k = lo; k < hi; k++) {
          const char* sp = operand(k);
#pragma unroll
          for (int u = 0; u < kUnroll; u++) {
            const size_t v = v0 + (size_t)u * nth;
            if (v < nv) cp_async16(&g_stage[((k - lo) * kUnroll + u) * nth + tid], sp + v * 16);
          }
        }
        cp_async_wait_all();
      }
      return j - lo;
    };
    A acc[kUnroll][V];
    uint4 pk[kUnroll];
    for (int s = 0; s < inner.n; s++) {  // ---- inner fold -> P_kpos (narrowed, kept packed) ----
      const int sl = stage(s);
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        const uint4 w = g_stage[(sl * kUnroll + u) * nth + tid];
#pragma unroll
        for (int e = 0; e < V; e++) {
          const A x = TR::widen(Vec<S>::get(w, e));
          acc[u][e] = s == 0 ? x : comb<OP>(acc[u][e], x);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int e = 0; e < V; e++) Vec<S>::set(pk[u], e, TR::narrow(acc[u][e]));
    for (int q = 0; q < D; q++) {  // ---- outer fold over the D domain partials in ascending order ----
      if (q == kpos) {
#pragma unroll
        for (int u = 0; u < kUnroll; u++)
#pragma unroll
          for (int e = 0; e < V; e++) {
            const A x = TR::widen(Vec<S>::get(pk[u], e));
            acc[u][e] = q == 0 ? x : comb<OP>(acc[u][e], x);
          }
        continue;
      }
      const int sl = stage(inner.n + (q < kpos ? q : q - 1));
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        const uint4 w = g_stage[(sl * kUnroll + u) * nth + tid];
#pragma unroll
        for (int e = 0; e < V; e++) {
          const A x = TR::widen(Vec<S>::get(w, e));
          acc[u][e] = q == 0 ? x : comb<OP>(acc[u][e], x);
        }
      }
    }
    uint4 o[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int e = 0; e < V; e++) Vec<S>::set(o[u], e, TR::narrow(acc[u][e]));
    for (int d = 0; d < dsts.n; d++) {
      char* dp = (char*)dsts.p[d];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        size_t v = v0 + (size_t)u * nth;
        if (v < nv) st_v4(dp + v * 16, o[u]);
      }
    }
  }
  } else {
  for (size_t v0 = tid; v0 < nvr; v0 += (size_t)kUnroll * nth) {
    for (int s = 0; s < inner.n; s++) prefetch_ahead(inner.p[s], v0, tid, (size_t)kUnroll * nth, nv);
    for (int q = 0; q < D; q++)
      if (q != kpos) prefetch_ahead(outer.p[q], v0, tid, (size_t)kUnroll * nth, nv);
    A acc[kUnroll][V];
    uint4 pk[kUnroll];
    // ---- inner fold -> P_kpos (narrowed, kept packed) ----
    for (int s = 0; s < inner.n; s++) {
      uint4 w[kUnroll];
      const char* sp = (const char*)inner.p[s];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        size_t v = v0 + (size_t)u * nth;
        if (v < nv) w[u] = ld_v4(sp + v * 16);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; u++)
#pragma unroll
        for (int e = 0; e < V; e++) {
          const A x = TR::widen(Vec<S>::get(w[u], e));
          acc[u][e] = s == 0 ? x : comb<OP>(acc[u][e], x);
        }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int e = 0; e < V; e++) Vec<S>::set(pk[u], e, TR::narrow(acc[u][e]));
    // ---- outer fold over the D domain partials in ascending order ----
    for (int q = 0; q < D; q++) {
      if (q == kpos) {
#pragma unroll
        for (int u = 0; u < kUnroll; u++)
#pragma unroll
          for (int e = 0; e < V; e++) {
            const A x = TR::widen(Vec<S>::get(pk[u], e));
            acc[u][e] = q == 0 ? x : comb<OP>(acc[u][e], x);
          }
        continue;
      }
      uint4 w[kUnroll];
      const char* sp = (const char*)outer.p[q];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        size_t v = v0 + (size_t)u * nth;
        if (v < nv) w[u] = ld_v4(sp + v * 16);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; u++)
#pragma unroll
        for (int e = 0; e < V; e++) {
          const A x = TR::widen(Vec<S>::get(w[u], e));
          acc[u][e] = q == 0 ? x : comb<OP>(acc[u][e], x);
        }
    }
    uint4 o[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int e = 0; e < V; e++) Vec<S>::set(o[u], e, TR::narrow(acc[u][e]));
    for (int d = 0; d < dsts.n; d++) {
      char* dp = (char*)dsts.p[d];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        size_t v = v0 + (size_t)u * nth;
        if (v < nv) st_v4(dp + v * 16, o[u]);
      }
    }
  }
  }
  for (size_t i = nv * V + tid; i < n; i += nth) {
    A a = 0;
    for (int s = 0; s < inner.n; s++) {
      S w = sizeof(S) == 4 ? (S)ld_s32((const char*)inner.p[s] + i * 4) : (S)ld_s16((const char*)inner.p[s] + i * 2);
      a = s == 0 ? TR::widen(w) : comb<OP>(a, TR::widen(w));
    }
    const S pks = TR::narrow(a);
    for (int q = 0; q < D; q++) {
      S w = q == kpos ? pks
                      : (sizeof(S) == 4 ? (S)ld_s32((const char*)outer.p[q] + i * 4)
                                        : (S)ld_s16((const char*)outer.p[q] + i * 2));
      a = q == 0 ? TR::widen(w) : comb<OP>(a, TR::widen(w));
    }
    S r = TR::narrow(a);
    for (int d = 0; d < dsts.n; d++) {
      if (sizeof(S) == 4) st_s32((char*)dsts.p[d] + i * 4, (uint32_t)r);
      else st_s16((char*)dsts.p[d] + i * 2, (uint16_t)r);
    }
  }
}

// Multi-level fold over ALL ranks in the oracle's order (readings R3, R5, R6): srcs[r] is rank r's
// operand; P_q = fold over domain q's members (ascending rank), narrowed iff D > 1; result = fold of
// the P_q in ascending domain id, narrowed. The one-shot All-Reduce's reduction.
template <typename T, int OP>
__device__ __forceinline__ void cta_fold_domains(const PtrList& srcs, const Topo& tp, const PtrList& dsts, size_t n) {
  using TR = Tr<T>;
  using S = typename TR::S;
  using A = typename TR::A;
  constexpr int V = TR::V;
  if (n == 0) return;
  const int tid = (int)threadIdx.x - g_dbase, nth = g_dnth;
  const size_t nv = all_aligned16(srcs, dsts) ? n / V : 0;
  const int D = tp.D;
  for (size_t v0 = tid; v0 < nv; v0 += (size_t)kUnroll * nth) {
    for (int s = 0; s < srcs.n; s++) prefetch_ahead(srcs.p[s], v0, tid, (size_t)kUnroll * nth, nv);
    A out[kUnroll][V], acc[kUnroll][V];
    for (int q = 0; q < D; q++) {
      const int d = tp.dom_size[q];
      for (int i = 0; i < d; i++) {
        uint4 w[kUnroll];
        const char* sp = (const char*)srcs.p[tp.members[tp.dom_first[q] + i]];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
          size_t v = v0 + (size_t)u * nth;
          if (v < nv) w[u] = ld_v4(sp + v * 16);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; u++)
#pragma unroll
          for (int e = 0; e < V; e++) {
            const A x = TR::widen(Vec<S>::get(w[u], e));
            acc[u][e] = i == 0 ? x : comb<OP>(acc[u][e], x);
          }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; u++)
#pragma unroll
        for (int e = 0; e < V; e++) {
          const A p = D > 1 ? TR::widen(TR::narrow(acc[u][e])) : acc[u][e];
          out[u][e] = q == 0 ? p : comb<OP>(out[u][e], p);
        }
    }
    uint4 o[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int e = 0; e < V; e++) Vec<S>::set(o[u], e, TR::narrow(out[u][e]));
    for (int d = 0; d < dsts.n; d++) {
      char* dp = (char*)dsts.p[d];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        size_t v = v0 + (size_t)u * nth;
        if (v < nv) st_v4(dp + v * 16, o[u]);
      }
    }
  }
  for (size_t i = nv * V + tid; i < n; i += nth) {
    A out = 0;
    for (int q = 0; q < D; q++) {
      A acc = 0;
      for (int k = 0; k < tp.dom_size[q]; k++) {
        const char* sp = (const char*)srcs.p[tp.members[tp.dom_first[q] + k]];
        S w = sizeof(S) == 4 ? (S)ld_s32(sp + i * 4) : (S)ld_s16(sp + i * 2);
        acc = k == 0 ? TR::widen(w) : comb<OP>(acc, TR::widen(w));
      }
      const A p = D > 1 ? TR::widen(TR::narrow(acc)) : acc;
      out = q == 0 ? p : comb<OP>(out, p);
    }
    S r = TR::narrow(out);
    for (int d = 0; d < dsts.n; d++) {
      if (sizeof(S) == 4) st_s32((char*)dsts.p[d] + i * 4, (uint32_t)r);
      else st_s16((char*)dsts.p[d] + i * 2, (uint16_t)r);
    }
  }
}

// ------------------------------------------------------------------ protocol helpers -----------
__device__ __forceinline__ uint64_t* chan_flags(const OpArgs& a, int rank, int ch) {
  return a.mem[rank].flags + (size_t)ch * kChanWords;
}
__device__ __forceinline__ uint64_t* chan_base(const OpArgs& a, int rank, int ch) {
  return (uint64_t*)((char*)a.mem[rank].flags + kFlagsReserve / 2) + (size_t)ch * kChanWords;
}

template <typename T>
__device__ __forceinline__ T* slot_ptr(const OpArgs& a, int rank, int ch, int slot) {
  return (T*)(a.mem[rank].scratch + ((size_t)ch * a.nslots + slot) * a.slot_elems * sizeof(T));
}

__device__ __forceinline__ size_t floor_to(size_t x, size_t q) { return x / q * q; }

// Elementary-segment and piece boundaries of one AR/BC tile (same formulas as plan.cpp): the grid
// of a FULL tile (segment = T/L, piece = T/(L*D) elements, multiples of the vector width because T
// is a multiple of L*D*V) clipped to the tile's length, so no piece of a ragged last tile is ever
// longer than its scratch slot.
struct Geo {
  size_t len, T;
  int L, D;
  __device__ size_t seg(int s) const { return min(len, (size_t)s * (T / L)); }
  __device__ size_t piece(int s, int p) const { return min(seg(s + 1), seg(s) + (size_t)p * (T / L / D)); }
};

// piece i of dd of a shard tile (RS / AG): full-tile grid T/dd clipped to len
__device__ __forceinline__ size_t sub_lo(size_t len, size_t T, int dd, int i) { return min(len, (size_t)i * (T / dd)); }

// compact index of domain member i in a buffer that has no entry for member j (the owner itself)
__device__ __forceinline__ int cidx(int i, int j) { return i < j ? i : i - 1; }

__device__ __forceinline__ int owner_of(const Topo& t, int q, int s) {
  return t.members[t.dom_first[q] + s / (t.L / t.dom_size[q])];
}

// ================================================================== pipeline driver ===========
// Software pipeline over the tiles t = ch, ch + nch, ... of one channel. The op's active logical
// stages occupy positions 0, SP, 2*SP, ... (identical on every rank); iteration `it` runs the stage at
// position p on the channel's local tile it - p. Warp 0 is the SYNC warp (polls, fences, signals);
// in the default warp-specialised mode (SP = 2) warps 1..15 move data while warp 0 releases the
// previous iteration, so the release fence (which waits for every outstanding NVLink store to be
// acknowledged) never stalls the data warps:
//   sync warp:  poll(0); for it: GO | fence; signal(it-1) | DONE | poll(it+1);  fence; signal(last)
//   data warps:          for it: GO | work(it)             | DONE
//   poll(it):   lane p polls sender p's counter of every stage due in iteration it (cumulative
//               target base + tile + 1) and, for position 0, the ACK of the tile that last used
//               the slot (nslots-deep ring);
//   signal(it): lane r adds 1 to rank r's counter for every stage of iteration it that signals r,
//               and after the last position's tile an ACK to every other rank.
// Because signal(it) is only sent during iteration it+1, a consumer sits SP = 2 positions after its
// producer: poll(it) then needs other ranks' signals of iterations <= it-2, sent in their window
// it-1, which needs their poll(it-1) — by induction no cycle, hence no deadlock with all CTAs
// co-resident. (HETCCL_WS=0 selects the plain mode: SP = 1, all 16 warps move data, and the sync
// warp fences and signals iteration it before polling it+1.)
struct PipeShared {
  unsigned long long base[kCounters][kMaxRanks];
  unsigned long long tiles0;
  int abort_;
};

template <class Op>
struct Pipe {
  const OpArgs& a;
  Op& op;
  PipeShared& ps;
  const RankPlan& rp;
  int me, ch, n, np, SP, npos, lane;
  long long ntl;
  unsigned long long tiles0;
  int stage_at[4 * kMaxStages];  // logical stage at each position, -1 for a bubble
  uint64_t* F;

  __device__ bool tile_at(long long it, int p, long long& tl) const {
    tl = it - p;
    return tl >= 0 && tl < ntl;
  }
  // sync warp: wait for everything iteration `it` needs; false on timeout
  // (position, sender) pairs are spread over the warp's lanes, so every counter of the iteration is read
  // in parallel (one flag round trip per iteration, not one per position)
  __device__ bool poll(long long it) {
    bool ok = true;
    for (int idx = lane; idx < npos * n && ok; idx += 32) {
      const int p = idx / n, snd = idx % n;
      long long tl;
      if (stage_at[p] < 0 || !tile_at(it, p, tl)) continue;
      const int s = stage_at[p];
      const uint64_t* w1 = nullptr;
      uint64_t t1 = 0;
      if (p == 0 && ((rp.writes >> snd) & 1u) && tiles0 + tl >= (unsigned long long)a.nslots) {
        w1 = F + C_ACK * kLineWords + snd;
        t1 = tiles0 + tl - a.nslots + 1;
      }
      const int wc = rp.wait_ctr[s];
      const uint64_t* w2 = nullptr;
      uint64_t t2 = 0;
      if (wc != C_NONE && ((rp.wait_mask[s] >> snd) & 1u)) {
        w2 = F + wc * kLineWords + snd;
        t2 = ps.base[wc][snd] + tl + 1;
      }
      for (int q = 0; q < 2 && ok; q++) {
        const uint64_t* w = q ? w2 : w1;
        const uint64_t tg = q ? t2 : t1;
        if (!w || ld_acquire(w, a.gpu_scope) >= tg) continue;
        const uint64_t t0 = globaltimer();
        uint32_t spins = 0;
        while (ld_acquire(w, a.gpu_scope) < tg) {
          if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > a.timeout_ns) {
            atomicOr(a.err, 1ull + ((unsigned long long)(q ? wc : C_ACK) << 8) + ((unsigned long long)snd << 16));
            ok = false;
            break;
          }
        }
      }
    }
    return ok;
  }
  // sync warp: every data store of iteration `it` is complete (caller fenced); signal its receivers
  __device__ void signal(long long it) {
    if (lane >= n || lane == me) return;
    int last = -1;
    for (int p = 0; p < npos; p++) {
      long long tl;
      if (stage_at[p] < 0) continue;
      last = p;
      if (!tile_at(it, p, tl)) continue;
      const int s = stage_at[p];
      if (rp.sig_ctr[s] != C_NONE && ((rp.sig_mask[s] >> lane) & 1u))
        red_add_relaxed(chan_flags(a, lane, ch) + rp.sig_ctr[s] * kLineWords + me, 1, a.gpu_scope);
    }
    long long tl;
    if (last >= 0 && tile_at(it, last, tl)) red_add_relaxed(chan_flags(a, lane, ch) + C_ACK * kLineWords + me, 1, a.gpu_scope);
  }
  unsigned long long* trc = nullptr;  // per-iteration stamps (HETCCL_TRACE_ITERS), thread 0 only
  // C stage of my tile t with chunk stealing (owner side); false if the job cannot be shared (several pieces)
  __device__ bool owner_c(size_t t, int slot, long long tl) {
    if constexpr (!Op::kSteal) {
      return false;
    } else {
      if (ntl != 1 || tl >= 4096 || slot >= 16 || op.c_pieces(t) != 1) return false;
      const int tid = (int)threadIdx.x - g_dbase;
      uint64_t* sw = chan_flags(a, me, ch) + (size_t)kCounters * kLineWords;
      if (tid == 0) {
        g_claim = sw;
        g_claim_mode = 1;
        g_claim_tag = ((uint64_t)tl << 52) | ((uint64_t)slot << 48);
        g_job_total = 0;
        g_claimed = 0;
      }
      data_bar();
      if (a.steal < 100) {  // the static part first, at full speed (bulk-copy stores, no claims)
        if (tid == 0) g_claim_mode = 0;
        data_bar();
        op.stage_c_part(t, slot, 0, a.steal);
        if (tid == 0) g_claim_mode = 1;
        data_bar();
      }
      op.stage_c_part(t, slot, 1, a.steal);  // its ring mover publishes the tail job and claims from the front
      data_bar();
      if (tid == 0) {
        g_claim_mode = 0;
        const uint64_t total = g_job_total, mine = g_claimed;
        const uint64_t t0 = globaltimer();
        uint32_t spins = 0;
        while (total > mine && ld_acquire_gpu(sw + 1) < total - mine) {  // the chunks other channels took
          if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > a.timeout_ns) {
            atomicOr(a.err, 1ull + ((unsigned long long)kCounters << 8) + ((unsigned long long)me << 16));
            ps.abort_ = 1;
            break;
          }
        }
      }
      data_bar();
      return true;
    }
  }
  // after my own pipeline: take chunks of the rank's other channels' published C stages. Thread 0 scans every
  // job word without a barrier and the data threads sync once per job found, so a CTA with nothing to take
  // leaves at once (a barrier per victim kept idle helpers around long enough to delay the kernel, r02bp).
  __device__ void help_others() {
    if constexpr (Op::kSteal) {
      const int tid = (int)threadIdx.x - g_dbase;
      __shared__ int s_victim;
      int start = 1;
      for (;;) {
        if (tid == 0) {
          s_victim = -1;
          for (int kk = start; kk < a.nch; kk++) {
            const int v = (ch + kk) % a.nch;
            uint64_t* sw = chan_flags(a, me, v) + (size_t)kCounters * kLineWords;
            const uint64_t w = ld_acquire_gpu(sw);
            if ((w & 0xffffffull) < ((w >> 24) & 0xffffffull)) {
              s_victim = kk;
              g_claim = sw;
              g_claim_mode = 2;
              g_claim_tag = w & kTagMask;
              g_claimed = 0;
              g_vec_only = 1;
              break;
            }
          }
        }
        data_bar();
        const int kk = s_victim;
        if (kk < 0) break;
        start = kk;  // the same victim may still have chunks; the scan moves on once it is exhausted
        const int v = (ch + kk) % a.nch;
        const uint64_t tag = g_claim_tag;
        Op vop(a, blockIdx.y, v);
        const size_t tv = (size_t)v + (size_t)(tag >> 52) * a.nch;
        vop.stage_c_part(tv, (int)((tag >> 48) & 15u), 1, a.steal);  // vector part of the victim's tail
        data_bar();
        if (tid == 0) {
          g_claim_mode = 0;
          g_vec_only = 0;
          if (g_claimed) {
            fence_acq_rel(a.gpu_scope);  // my stores (peers' y included) before the owner's acquire
            red_add_relaxed(g_claim + 1, g_claimed, 1);
          }
        }
        data_bar();
      }
      if (tid == 0) {
        g_claim_mode = 0;
        g_vec_only = 0;
      }
    }
  }
  __device__ void work(long long it) {
    for (int p = 0; p < npos; p++) {
      long long tl;
      if (stage_at[p] < 0 || !tile_at(it, p, tl)) continue;
      if (a.steal && stage_at[p] == 2 &&
          owner_c((size_t)ch + (size_t)tl * a.nch, (int)((tiles0 + tl) % (unsigned long long)a.nslots), tl)) {
        if (trc && threadIdx.x == 0 && it < a.trace_iters) trc[it * kTraceWords + 4 + 2] = globaltimer();
        continue;
      }
      op.stage(stage_at[p], (size_t)ch + (size_t)tl * a.nch, (int)((tiles0 + tl) % (unsigned long long)a.nslots));
      if (trc && threadIdx.x == 0 && it < a.trace_iters && stage_at[p] < 4)
        trc[it * kTraceWords + 4 + stage_at[p]] = globaltimer();
    }
  }
};

template <class Op>
__device__ __forceinline__ void run_pipeline(const OpArgs& a, Op& op, int me, int ch) {
  const unsigned long long t_entry = globaltimer();
  __shared__ PipeShared ps;
  Pipe<Op> P{a, op, ps, a.rp[me]};
  P.me = me;
  P.ch = ch;
  P.n = a.topo.n;
  P.lane = threadIdx.x & 31;
  P.F = chan_flags(a, me, ch);
  uint64_t* B = chan_base(a, me, ch);
  const bool ws = a.ws >= 2;
  P.SP = ws ? a.ws : (a.spacing > 1 ? a.spacing : 1);  // plain mode: consumer positions SP apart (slack)
  P.np = 0;
  for (int p = 0; p < 4 * kMaxStages; p++) P.stage_at[p] = -1;
#pragma unroll
  for (int s = 0; s < kMaxStages; s++)
    if (((a.active >> s) & 1u) && s != a.final_stage) P.stage_at[P.SP * P.np++] = s;
  P.npos = P.SP * (P.np - 1) + 1;
  if (threadIdx.x < kCounters * kMaxRanks)
    ps.base[threadIdx.x / kMaxRanks][threadIdx.x % kMaxRanks] = B[threadIdx.x / kMaxRanks * kLineWords + threadIdx.x % kMaxRanks];
  tma_init(a.tma, (a.ws >= 2 ? (int)blockDim.x - 32 : (int)blockDim.x) / 32, a.l2hint, a.s2g);
  if (threadIdx.x == 0) {
    g_claim_mode = 0;
    g_vec_only = 0;
    ps.tiles0 = B[kCounters * kLineWords];
    ps.abort_ = 0;
    g_pf = !a.remote_pull;
    g_dbase = ws ? 32 : 0;
    g_dnth = ws ? (int)blockDim.x - 32 : (int)blockDim.x;
  }
  __syncthreads();
  P.ntl = (ch < (long long)a.ntiles) ? ((long long)a.ntiles - ch + a.nch - 1) / a.nch : 0;
  P.tiles0 = ps.tiles0;
  const long long nit = P.ntl > 0 ? P.ntl + P.npos - 1 : 0;
  // pull mode: my domain peers read my send buffer directly, so they must not start before it is ready
  // (this op started here): one release-signal / acquire-wait round per channel on counter S1
  if (a.pull && P.ntl > 0) {
    if (threadIdx.x < 32) {
      const Topo& tp = a.topo;
      const int k = tp.rank_dom[me];
      const bool dpeer = P.lane < P.n && P.lane != me && tp.rank_dom[P.lane] == k;
      fence_acq_rel(a.gpu_scope);
      if (dpeer) red_add_relaxed(chan_flags(a, P.lane, ch) + C_S1 * kLineWords + me, 1, a.gpu_scope);
      if (dpeer) {
        const uint64_t* w = P.F + C_S1 * kLineWords + P.lane;
        const uint64_t tg = ps.base[C_S1][P.lane] + 1;
        const uint64_t t0 = globaltimer();
        uint32_t spins = 0;
        while (ld_acquire(w, a.gpu_scope) < tg) {
          if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > a.timeout_ns) {
            atomicOr(a.err, 1ull + ((unsigned long long)C_S1 << 8) + ((unsigned long long)P.lane << 16));
            ps.abort_ = 1;
            break;
          }
        }
      }
    }
    __syncthreads();
  }
  const bool sync_warp = threadIdx.x < 32;
  unsigned long long* trc = nullptr;  // [it][kTraceWords] globaltimer stamps: poll start, GO, DONE, fenced, stage ends
  if (a.trace) trc = a.trace + ((size_t)blockIdx.y * gridDim.x + ch) * (size_t)a.trace_iters * kTraceWords;
  P.trc = trc;
  auto stamp = [&](long long it, int k) {
    if (trc && threadIdx.x == 0 && it >= 0 && it < a.trace_iters) trc[it * kTraceWords + k] = globaltimer();
  };
  if (ws) {
    if (sync_warp && nit > 0) {
      stamp(0, 0);
      if (!P.poll(0)) ps.abort_ = 1;
    }
    for (long long it = 0; it < nit; ++it) {
      __syncthreads();  // GO(it)
      if (*(volatile int*)&ps.abort_) break;
      stamp(it, 1);
      if (sync_warp) {
        if (it > 0) {
          fence_acq_rel(a.gpu_scope);
          stamp(it - 1, 3);
          P.signal(it - 1);
        }
      } else {
        P.work(it);
      }
      __syncthreads();  // DONE(it)
      stamp(it, 2);
      if (sync_warp && it + 1 < nit) {
        stamp(it + 1, 0);
        if (!P.poll(it + 1)) ps.abort_ = 1;
      }
    }
    if (sync_warp && nit > 0 && !*(volatile int*)&ps.abort_) {
      fence_acq_rel(a.gpu_scope);
      stamp(nit - 1, 3);
      P.signal(nit - 1);
    }
  } else {
    for (long long it = 0; it < nit; ++it) {
      stamp(it, 0);
      if (sync_warp && !P.poll(it)) ps.abort_ = 1;
      __syncthreads();
      if (*(volatile int*)&ps.abort_) break;
      stamp(it, 1);
      P.work(it);
      __syncthreads();
      stamp(it, 2);
      if (sync_warp) {
        fence_acq_rel(a.gpu_scope);
        stamp(it, 3);
        P.signal(it);
      }
    }
  }
  // ---- help the rank's other channels with their published C stages (HETCCL_STEAL) ----
  if (a.steal && a.steal_help && !*(volatile int*)&ps.abort_ && !(ws && sync_warp)) P.help_others();
  __syncthreads();
  // ---- final stage (direct All-Reduce's E): one wait for every tile's signal instead of a position ----
  if (a.final_stage >= 0 && ((a.active >> a.final_stage) & 1u) && threadIdx.x < 32 && P.lane < P.n &&
      !*(volatile int*)&ps.abort_) {
    const RankPlan& rp = a.rp[me];
    const int wc = rp.wait_ctr[a.final_stage];
    if (wc != C_NONE && ((rp.wait_mask[a.final_stage] >> P.lane) & 1u)) {
      const uint64_t* w = P.F + wc * kLineWords + P.lane;
      const uint64_t tg = ps.base[wc][P.lane] + P.ntl;
      const uint64_t t0 = globaltimer();
      uint32_t spins = 0;
      while (ld_acquire(w, a.gpu_scope) < tg) {
        if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > a.timeout_ns) {
          atomicOr(a.err, 1ull + ((unsigned long long)wc << 8) + ((unsigned long long)P.lane << 16));
          ps.abort_ = 1;
          break;
        }
      }
    }
  }
  __syncthreads();
  if (trc && threadIdx.x == 0) {
    trc[8] = t_entry;
    trc[9] = globaltimer();
  }
  // ---- exit: advance this rank's cumulative targets by the tiles this launch processed ----
  if (!ps.abort_ && threadIdx.x < kMaxRanks) {
    const int p = threadIdx.x;
    const RankPlan& rp = a.rp[me];
    for (int s = 0; s < kMaxStages; s++) {
      if (!((a.active >> s) & 1u)) continue;
      const int wc = rp.wait_ctr[s];
      if (wc != C_NONE && ((rp.wait_mask[s] >> p) & 1u)) B[wc * kLineWords + p] = ps.base[wc][p] + P.ntl;
    }
    if (p == 0) B[kCounters * kLineWords] = P.tiles0 + P.ntl;
    if (a.pull && P.ntl > 0 && p < P.n && p != me && a.topo.rank_dom[p] == a.topo.rank_dom[me])
      B[C_S1 * kLineWords + p] = ps.base[C_S1][p] + 1;  // the start round
  }
}

// ================================================================== All-Reduce (a1-a5) =========
// Slot layout on a rank of domain k (d = d_k, Rk = tile/d; s1/s3 have one entry per domain PEER,
// compact index cidx(i, j)):
//   s1[d-1][Rk] | s2[D][Rk] | ag[Rk] | s3[d-1][Rk]
// Stages: 0 A intra push | 1 B domain fold of the other domains' pieces + cross push |
//         2 C domain fold of my pieces + cross fold -> y, other owners' ag, domain peers' s3 |
//         3 D other owners' pieces (ag) -> y and domain peers | 4 E domain peers' regions -> y
template <typename T, int OP>
struct ArOp {
  static constexpr int ES = sizeof(T);
  static constexpr int V = Tr<T>::V;
  const OpArgs& a;
  const Topo& tp;
  int me, ch, k, j, d, D, L, spj, s_lo, s_hi;
  size_t TL, Rk;
  const T* x;
  T* y;
  __device__ ArOp(const OpArgs& a_, int row, int ch_) : a(a_), tp(a_.topo), ch(ch_) {
    me = a.local_rank[row];
    k = tp.rank_dom[me];
    j = tp.rank_idx[me];
    d = tp.dom_size[k];
    D = tp.D;
    L = tp.L;
    spj = L / d;
    s_lo = j * spj;
    s_hi = s_lo + spj;
    TL = a.tile;
    Rk = TL / d;
    x = (const T*)a.send[row];
    y = (T*)a.recv[row];
  }
  __device__ int peer(int i) const { return tp.members[tp.dom_first[k] + i]; }
  // offset of s2 in the slot of a rank whose domain has dq members
  __device__ size_t s2_off(int dq) const { return (size_t)(dq - 1) * (TL / dq); }
  // domain peer i's data for tile offset c (in my region): its send buffer (pull) or my s1 slot (push)
  __device__ const void* dsrc(int i, int slot, size_t tb, size_t c, size_t r0) const {
    if (a.pull) return (const T*)a.peer_send[peer(i)] + tb + c;
    return slot_ptr<T>(a, me, ch, slot) + (size_t)cidx(i, j) * Rk + (c - r0);
  }
  // start of the region of owner o (domain q) within a tile, and o's Rk
  __device__ size_t region_lo(const Geo& g, int o) const {
    const int q = tp.rank_dom[o];
    return g.seg(tp.rank_idx[o] * (L / tp.dom_size[q]));
  }
  // stage C on elements [c0, c1) of my piece of segment sg (any sub-range of the piece: every operand and
  // destination address is linear in the element offset)
  __device__ void fold_c(const Geo& g, int sg, size_t tb, size_t c0, size_t c1, int slot, size_t r0, T* my_s2) {
    PtrList inner, outer, dst;
    for (int i = 0; i < d; i++) inner.add(i == j ? (const void*)(x + tb + c0) : dsrc(i, slot, tb, c0, r0));
    for (int q = 0; q < D; q++) {
      if (q == k) outer.add(nullptr);
      else outer.add_keep(my_s2 + (size_t)q * Rk + (c0 - r0));  // dead after this read
    }
    dst.add(y + tb + c0);
    for (int q = 0; q < D; q++) {
      if (q == k) continue;
      const int o = owner_of(tp, q, sg);
      const int dq = tp.dom_size[q];
      if (a.flat_ag) {  // every member of domain q, not only the segment's owner (no forwarding stage D)
        for (int i = 0; i < dq; i++) dst.add((T*)a.peer_recv[tp.members[tp.dom_first[q] + i]] + tb + c0);
        continue;
      }
      if (a.direct) dst.add((T*)a.peer_recv[o] + tb + c0);  // straight into the owner's recv buffer
      else dst.add(slot_ptr<T>(a, o, ch, slot) + s2_off(dq) + (size_t)D * (TL / dq) + (c0 - region_lo(g, o)));
    }
    for (int i = 0; i < d; i++)
      if (i != j) {
        if (a.direct) dst.add((T*)a.peer_recv[peer(i)] + tb + c0);
        else
          dst.add(slot_ptr<T>(a, peer(i), ch, slot) + s2_off(d) + (size_t)(D + 1) * Rk + (size_t)cidx(j, i) * Rk +
                  (c0 - r0));
      }
    cta_fold_hier<T, OP>(inner, k, outer, dst, c1 - c0);
  }
  // number of non-empty pieces of my C stage in tile t (chunk stealing needs exactly one)
  __device__ int c_pieces(size_t t) const {
    const size_t tb = t * TL, len = min(TL, a.count - tb);
    const Geo g{len, TL, L, D};
    int np = 0;
    for (int sg = s_lo; sg < s_hi; sg++) np += g.piece(sg, k + 1) > g.piece(sg, k);
    return np;
  }
  // stage C of tile t (single piece) split at a 64-element boundary: part 0 = the first (100 - tail_pct)% run
  // statically by the owner, part 1 = the tail it publishes for chunk stealing (tail_pct = 100: all of it)
  __device__ void stage_c_part(size_t t, int slot, int part, int tail_pct) {
    const size_t tb = t * TL, len = min(TL, a.count - tb);
    const Geo g{len, TL, L, D};
    const size_t r0 = g.seg(s_lo);
    T* my_s2 = slot_ptr<T>(a, me, ch, slot) + s2_off(d);
    for (int sg = s_lo; sg < s_hi; sg++) {
      const size_t c0 = g.piece(sg, k), c1 = g.piece(sg, k + 1);
      if (c1 <= c0) continue;
      const size_t tail = min(c1 - c0, ((c1 - c0) * (size_t)tail_pct / 100 + 63) / 64 * 64);
      const size_t cm = c1 - tail;
      if (part == 0 && cm > c0) fold_c(g, sg, tb, c0, cm, slot, r0, my_s2);
      if (part == 1 && c1 > cm) fold_c(g, sg, tb, cm, c1, slot, r0, my_s2);
    }
  }
  static constexpr bool kSteal = true;  // stage 2 can be split into units other channels may take
  __device__ void stage(int s, size_t t, int slot) {
    const size_t tb = t * TL, len = min(TL, a.count - tb);
    const Geo g{len, TL, L, D};
    const size_t r0 = g.seg(s_lo), r1 = g.seg(s_hi);
    T* mine = slot_ptr<T>(a, me, ch, slot);
    T* my_s2 = mine + s2_off(d);
    T* my_ag = my_s2 + (size_t)D * Rk;
    T* my_s3 = my_ag + Rk;
    if (s == 0) {  // ---- A: push my data for each domain peer's region to its s1[j] ----
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const size_t p0 = g.seg(i * spj), p1 = g.seg((i + 1) * spj);
        cta_copy1<ES>(x + tb + p0, slot_ptr<T>(a, peer(i), ch, slot) + (size_t)cidx(j, i) * Rk, p1 - p0);
      }
    } else if (s == 1) {  // ---- B: fold the other domains' pieces of my region; push to their reducers ----
      for (int sg = s_lo; sg < s_hi; sg++) {
        for (int q = 0; q < D; q++) {
          if (D > 1 && q == k) continue;  // my own piece is folded in C (its partial never leaves registers)
          const size_t c0 = g.piece(sg, q), c1 = g.piece(sg, q + 1);
          if (c1 <= c0) continue;
          PtrList src, dst;
          for (int i = 0; i < d; i++)
            src.add(i == j ? (const void*)(x + tb + c0) : dsrc(i, slot, tb, c0, r0));
          if (D == 1) {
            dst.add(y + tb + c0);
          } else {
            const int o = owner_of(tp, q, sg);
            const int dq = tp.dom_size[q];
            dst.add_keep(slot_ptr<T>(a, o, ch, slot) + s2_off(dq) + (size_t)k * (TL / dq) + (c0 - region_lo(g, o)));
          }
          cta_fold<T, OP>(src, dst, c1 - c0);
        }
      }
    } else if (s == 2) {  // ---- C: P_k of my pieces (domain fold) + the other partials; final -> y, owners, peers ----
      for (int sg = s_lo; sg < s_hi; sg++) {
        const size_t c0 = g.piece(sg, k), c1 = g.piece(sg, k + 1);
        if (c1 > c0) fold_c(g, sg, tb, c0, c1, slot, r0, my_s2);
      }
    } else if (s == 3 && a.direct) {  // ---- D (direct): forward the other owners' pieces (now in y) to peers ----
      PtrList peers_y;
      for (int i = 0; i < d; i++)
        if (i != j) peers_y.add((T*)a.peer_recv[peer(i)] + tb);
      if (!peers_y.n) return;
      if (D == 1) {
        PtrList dst;
        for (int i = 0; i < peers_y.n; i++) dst.add((const char*)peers_y.p[i] + r0 * ES);
        cta_copy<ES>(y + tb + r0, dst, r1 - r0);
      } else {
        for (int sg = s_lo; sg < s_hi; sg++)
          for (int q = 0; q < D; q++) {
            if (q == k) continue;
            const size_t c0 = g.piece(sg, q), c1 = g.piece(sg, q + 1);
            if (c1 <= c0) continue;
            PtrList dst;
            for (int i = 0; i < peers_y.n; i++) dst.add((const char*)peers_y.p[i] + c0 * ES);
            cta_copy<ES>(y + tb + c0, dst, c1 - c0);
          }
      }
    } else if (s == 4 && a.direct) {  // ---- E (direct): nothing to copy; the S3 wait made y complete ----
      return;
    } else if (s == 3) {  // ---- D: the other owners' final pieces of my region -> y and domain peers ----
      PtrList peers_s3;
      for (int i = 0; i < d; i++)
        if (i != j) peers_s3.add(slot_ptr<T>(a, peer(i), ch, slot) + s2_off(d) + (size_t)(D + 1) * Rk + (size_t)cidx(j, i) * Rk);
      if (D == 1) {
        cta_copy<ES>(y + tb + r0, peers_s3, r1 - r0);
      } else {
        for (int sg = s_lo; sg < s_hi; sg++) {
          for (int q = 0; q < D; q++) {
            if (q == k) continue;  // pushed to the peers by C
            const size_t c0 = g.piece(sg, q), c1 = g.piece(sg, q + 1);
            if (c1 <= c0) continue;
            PtrList dst;
            dst.add(y + tb + c0);
            for (int i = 0; i < peers_s3.n; i++) dst.add((const char*)peers_s3.p[i] + (c0 - r0) * ES);
            cta_copy<ES>(my_ag + (c0 - r0), dst, c1 - c0);
          }
        }
      }
    } else {  // ---- E: domain peers' final regions -> y ----
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const size_t p0 = g.seg(i * spj), p1 = g.seg((i + 1) * spj);
        cta_copy1<ES>(my_s3 + (size_t)cidx(i, j) * Rk, y + tb + p0, p1 - p0);
      }
    }
  }
};

// ================================================================== Reduce-Scatter (a6) ========
// Per tile (per-shard offsets [tb, tb+len)), member j of domain k owns: its own shard, plus piece j
// (of d) of every other-domain shard. Slot layout on a rank of domain k (RG = T + (n-d)*T/d):
//   s1[d-1][RG] | s2[D][T]  (s1[cidx(i,j)]: own-shard part at 0, other-domain shard #ro at T + ro*T/d)
// Stages: 0 A intra push | 1 B domain fold of other shards' pieces + cross push |
//         2 C domain fold of my shard + cross fold -> y
template <typename T, int OP>
struct RsOp {
  static constexpr bool kSteal = false;
  static constexpr int ES = sizeof(T);
  static constexpr int V = Tr<T>::V;
  const OpArgs& a;
  const Topo& tp;
  int me, ch, n, k, j, d, D;
  size_t TL, R, Pc, RG;
  const T* x;
  T* y;
  __device__ RsOp(const OpArgs& a_, int row, int ch_) : a(a_), tp(a_.topo), ch(ch_) {
    me = a.local_rank[row];
    n = tp.n;
    k = tp.rank_dom[me];
    j = tp.rank_idx[me];
    d = tp.dom_size[k];
    D = tp.D;
    TL = a.tile;
    R = a.count;
    Pc = TL / d;
    RG = TL + (size_t)(n - d) * Pc;
    x = (const T*)a.send[row];
    y = (T*)a.recv[row];
  }
  __device__ void stage(int s, size_t t, int slot) {
    const size_t tb = t * TL, len = min(TL, R - tb);
    T* mine = slot_ptr<T>(a, me, ch, slot);
    const size_t pj0 = sub_lo(len, TL, d, j), pj1 = sub_lo(len, TL, d, j + 1);
    if (s == 0) {  // ---- A: each domain peer gets my data for its region ----
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const int pr = tp.members[tp.dom_first[k] + i];
        T* dst = slot_ptr<T>(a, pr, ch, slot) + (size_t)cidx(j, i) * RG;
        cta_copy1<ES>(x + (size_t)pr * R + tb, dst, len);
        const size_t pi0 = sub_lo(len, TL, d, i), pi1 = sub_lo(len, TL, d, i + 1);
        int ro = 0;
        for (int r = 0; r < n; r++) {
          if (tp.rank_dom[r] == k) continue;
          cta_copy1<ES>(x + (size_t)r * R + tb + pi0, dst + TL + (size_t)ro * Pc, pi1 - pi0);
          ro++;
        }
      }
    } else if (s == 1) {  // ---- B: own shard -> domain partial; my pieces of other shards -> their owners ----
      if (D == 1) {  // one domain: the domain fold is the result (with D > 1 it is folded in C)
        PtrList src, dst;
        for (int i = 0; i < d; i++)
          src.add(i == j ? (const void*)(x + (size_t)me * R + tb) : (const void*)(mine + (size_t)cidx(i, j) * RG));
        dst.add(y + tb);
        cta_fold<T, OP>(src, dst, len);
      }
      int ro = 0;
      for (int r = 0; r < n; r++) {
        if (tp.rank_dom[r] == k) continue;
        PtrList src, dst;
        for (int i = 0; i < d; i++)
          src.add(i == j ? (const void*)(x + (size_t)r * R + tb + pj0)
                         : (const void*)(mine + (size_t)cidx(i, j) * RG + TL + (size_t)ro * Pc));
        const int dr = tp.dom_size[tp.rank_dom[r]];
        const size_t RGr = TL + (size_t)(n - dr) * (TL / dr);
        dst.add_keep(slot_ptr<T>(a, r, ch, slot) + (size_t)(dr - 1) * RGr + (size_t)k * TL + pj0);
        cta_fold<T, OP>(src, dst, pj1 - pj0);
        ro++;
      }
    } else {  // ---- C: my domain's partial of my shard + the D-1 others (ascending domain id) -> y ----
      PtrList inner, outer, dst;
      for (int i = 0; i < d; i++)
        inner.add(i == j ? (const void*)(x + (size_t)me * R + tb) : (const void*)(mine + (size_t)cidx(i, j) * RG));
      for (int q = 0; q < D; q++) {
        if (q == k) outer.add(nullptr);
        else outer.add_keep(mine + (size_t)(d - 1) * RG + (size_t)q * TL);  // dead after this read
      }
      dst.add(y + tb);
      cta_fold_hier<T, OP>(inner, k, outer, dst, len);
    }
  }
};

// ================================================================== All-Gather (a7) ============
// Mirror of reduce-scatter. Slot layout on a rank of domain k (RG = T + (n-d)*T/d):
//   s_in[d-1][RG] | xin[n-d][T/d]
// Stages: 0 A cross push | 1 B own shard + received pieces -> y and domain peers | 2 C peers -> y
template <typename T>
struct AgOp {
  static constexpr bool kSteal = false;
  static constexpr int ES = sizeof(T);
  static constexpr int V = 16 / ES;
  const OpArgs& a;
  const Topo& tp;
  int me, ch, n, k, j, d, D;
  size_t TL, R, Pc, RG;
  const T* x;
  T* y;
  bool inplace;
  __device__ AgOp(const OpArgs& a_, int row, int ch_) : a(a_), tp(a_.topo), ch(ch_) {
    me = a.local_rank[row];
    n = tp.n;
    k = tp.rank_dom[me];
    j = tp.rank_idx[me];
    d = tp.dom_size[k];
    D = tp.D;
    TL = a.tile;
    R = a.count;
    Pc = TL / d;
    RG = TL + (size_t)(n - d) * Pc;
    x = (const T*)a.send[row];
    y = (T*)a.recv[row];
    inplace = (x == y + (size_t)me * R);
  }
  __device__ int peer(int i) const { return tp.members[tp.dom_first[k] + i]; }
  __device__ void stage(int s, size_t t, int slot) {
    const size_t tb = t * TL, len = min(TL, R - tb);
    T* mine = slot_ptr<T>(a, me, ch, slot);
    T* xin = mine + (size_t)(d - 1) * RG;
    const size_t pj0 = sub_lo(len, TL, d, j), pj1 = sub_lo(len, TL, d, j + 1);
    if (s == 0) {  // ---- A: piece i of my shard to member i of every other domain ----
      for (int r = 0; r < n; r++) {
        const int q = tp.rank_dom[r];
        if (q == k) continue;
        const int dq = tp.dom_size[q], i = tp.rank_idx[r];
        int ro_me = 0;  // my index among the ranks outside domain q
        for (int r2 = 0; r2 < me; r2++)
          if (tp.rank_dom[r2] != q) ro_me++;
        const size_t a0 = sub_lo(len, TL, dq, i), a1 = sub_lo(len, TL, dq, i + 1);
        const size_t RGq = TL + (size_t)(n - dq) * (TL / dq);
        cta_copy1<ES>(x + tb + a0, slot_ptr<T>(a, r, ch, slot) + (size_t)(dq - 1) * RGq + (size_t)ro_me * (TL / dq), a1 - a0);
      }
    } else if (s == 1) {  // ---- B: my region (own shard + received pieces) -> y and every domain peer ----
      PtrList dst_shard;
      if (!inplace) dst_shard.add(y + (size_t)me * R + tb);
      for (int i = 0; i < d; i++)
        if (i != j) dst_shard.add(slot_ptr<T>(a, peer(i), ch, slot) + (size_t)cidx(j, i) * RG);
      if (dst_shard.n) cta_copy<ES>(x + tb, dst_shard, len);
      int ro = 0;
      for (int r = 0; r < n; r++) {
        if (tp.rank_dom[r] == k) continue;
        PtrList dst;
        dst.add(y + (size_t)r * R + tb + pj0);
        for (int i = 0; i < d; i++)
          if (i != j) dst.add(slot_ptr<T>(a, peer(i), ch, slot) + (size_t)cidx(j, i) * RG + TL + (size_t)ro * Pc);
        cta_copy<ES>(xin + (size_t)ro * Pc, dst, pj1 - pj0);
        ro++;
      }
    } else {  // ---- C: every domain peer's region -> y ----
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const int pr = peer(i);
        const T* reg = mine + (size_t)cidx(i, j) * RG;
        cta_copy1<ES>(reg, y + (size_t)pr * R + tb, len);
        const size_t pi0 = sub_lo(len, TL, d, i), pi1 = sub_lo(len, TL, d, i + 1);
        int ro = 0;
        for (int r = 0; r < n; r++) {
          if (tp.rank_dom[r] == k) continue;
          cta_copy1<ES>(reg + TL + (size_t)ro * Pc, y + (size_t)r * R + tb + pi0, pi1 - pi0);
          ro++;
        }
      }
    }
  }
};

// ================================================================== Broadcast (a8) =============
// Root -> its domain members (scatter of regions) -> one owner per other domain per segment ->
// intra-domain all-gather. Slot layout on a rank of domain k (Rk = T/d): reg[Rk] | s3[d-1][Rk]
// Stages: 0 A root scatter | 1 B cross push | 2 C region -> y and domain peers | 3 D peers -> y
template <typename T>
struct BcOp {
  static constexpr bool kSteal = false;
  static constexpr int ES = sizeof(T);
  static constexpr int V = 16 / ES;
  const OpArgs& a;
  const Topo& tp;
  int me, ch, k, j, d, D, L, spj, s_lo, s_hi, root, kr;
  size_t TL, Rk;
  const T* x;
  T* y;
  bool is_root;
  __device__ BcOp(const OpArgs& a_, int row, int ch_) : a(a_), tp(a_.topo), ch(ch_) {
    me = a.local_rank[row];
    k = tp.rank_dom[me];
    j = tp.rank_idx[me];
    d = tp.dom_size[k];
    D = tp.D;
    L = tp.L;
    spj = L / d;
    s_lo = j * spj;
    s_hi = s_lo + spj;
    root = a.root;
    kr = tp.rank_dom[root];
    TL = a.tile;
    Rk = TL / d;
    x = (const T*)a.send[row];
    y = (T*)a.recv[row];
    is_root = (me == root);
  }
  __device__ int peer(int i) const { return tp.members[tp.dom_first[k] + i]; }
  // the member of the root's domain that takes over the root's region (plan.cpp bcast_relay), or -1
  __device__ int relay() const {
    const int dr = tp.dom_size[kr];
    return dr < 2 ? -1 : tp.members[tp.dom_first[kr] + (tp.rank_idx[root] + 1) % dr];
  }
  __device__ void stage(int s, size_t t, int slot) {
    const size_t tb = t * TL, len = min(TL, a.count - tb);
    const Geo g{len, TL, L, 1};
    T* mine = slot_ptr<T>(a, me, ch, slot);
    const size_t r0 = g.seg(s_lo), r1 = g.seg(s_hi);
    const T* myreg = is_root ? (x + tb + r0) : mine;
    const int rl = relay(), rj = tp.rank_idx[root];
    const bool am_relay = (me == rl);
    // the root's region as the relay holds it: my s3 entry for the root (filled by the root in A)
    const T* rootreg = am_relay ? mine + Rk + (size_t)cidx(rj, j) * Rk : nullptr;
    const size_t q0 = g.seg(rj * spj), q1 = g.seg((rj + 1) * spj);  // root's region (in its domain)
    if (s == 0) {  // ---- A: the root scatters the regions of its domain (its own to the relay) ----
      if (!is_root) return;
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const size_t p0 = g.seg(i * spj), p1 = g.seg((i + 1) * spj);
        cta_copy1<ES>(x + tb + p0, slot_ptr<T>(a, peer(i), ch, slot), p1 - p0);
        if (peer(i) == rl) cta_copy1<ES>(x + tb + r0, slot_ptr<T>(a, rl, ch, slot) + Rk + (size_t)cidx(j, i) * Rk, r1 - r0);
      }
    } else if (s == 1) {  // ---- B: each root-domain segment to its owner in every other domain ----
      if (k != kr || (is_root && rl >= 0)) return;
      for (int pass = 0; pass < (am_relay ? 2 : 1); pass++) {
        const int lo = pass ? rj * spj : s_lo, hi = pass ? (rj + 1) * spj : s_hi;
        const T* src = pass ? rootreg : myreg;
        const size_t base = pass ? q0 : r0;
        for (int sg = lo; sg < hi; sg++) {
          const size_t c0 = g.seg(sg), c1 = g.seg(sg + 1);
          PtrList dst;
          for (int q = 0; q < D; q++) {
            if (q == kr) continue;
            const int o = owner_of(tp, q, sg);
            const size_t ro = g.seg(tp.rank_idx[o] * (L / tp.dom_size[q]));
            dst.add(slot_ptr<T>(a, o, ch, slot) + (c0 - ro));
          }
          cta_copy<ES>(src + (c0 - base), dst, c1 - c0);
        }
      }
    } else if (s == 2) {  // ---- C: my region (and the relay: the root's) -> y and every peer but the root ----
      if (is_root) {
        if (x != y) cta_copy1<ES>(x + tb, y + tb, len);
        return;
      }
      PtrList dst;
      dst.add(y + tb + r0);
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const int pr = peer(i);
        if (pr == root) continue;
        dst.add(slot_ptr<T>(a, pr, ch, slot) + Rk + (size_t)cidx(j, i) * Rk);
      }
      cta_copy<ES>(myreg, dst, r1 - r0);
      if (am_relay) {
        PtrList dr;
        dr.add(y + tb + q0);
        for (int i = 0; i < d; i++) {
          if (i == j) continue;
          const int pr = peer(i);
          if (pr == root) continue;
          dr.add(slot_ptr<T>(a, pr, ch, slot) + Rk + (size_t)cidx(rj, i) * Rk);
        }
        cta_copy<ES>(rootreg, dr, q1 - q0);
      }
    } else {  // ---- D: domain peers' regions (the root's via the relay) -> y ----
      if (is_root) return;
      for (int i = 0; i < d; i++) {
        if (i == j || (am_relay && i == rj && k == kr)) continue;
        const size_t p0 = g.seg(i * spj), p1 = g.seg((i + 1) * spj);
        cta_copy1<ES>(mine + Rk + (size_t)cidx(i, j) * Rk, y + tb + p0, p1 - p0);
      }
    }
  }
};

// ================================================================== Reduce (NEXT-2) =============
// out_root = the All-Reduce result Y (same fold order). Stages A/B as All-Reduce; C folds my pieces with
// the other domains' partials (cta_fold_hier) and sends the final piece to the root; D: the root copies
// everyone's pieces into y. Slot layout on a rank of domain k: s1[d-1][Rk] | s2[D][Rk] | fin[T] (root).
template <typename T, int OP>
struct RdOp {
  static constexpr bool kSteal = false;
  static constexpr int ES = sizeof(T);
  const OpArgs& a;
  const Topo& tp;
  int me, ch, k, j, d, D, L, spj, s_lo, s_hi, root;
  size_t TL, Rk;
  const T* x;
  T* y;
  __device__ RdOp(const OpArgs& a_, int row, int ch_) : a(a_), tp(a_.topo), ch(ch_) {
    me = a.local_rank[row];
    k = tp.rank_dom[me];
    j = tp.rank_idx[me];
    d = tp.dom_size[k];
    D = tp.D;
    L = tp.L;
    spj = L / d;
    s_lo = j * spj;
    s_hi = s_lo + spj;
    root = a.root;
    TL = a.tile;
    Rk = TL / d;
    x = (const T*)a.send[row];
    y = (T*)a.recv[row];
  }
  __device__ int peer(int i) const { return tp.members[tp.dom_first[k] + i]; }
  __device__ size_t s2_off(int dq) const { return (size_t)(dq - 1) * (TL / dq); }
  __device__ size_t region_lo(const Geo& g, int o) const {
    const int q = tp.rank_dom[o];
    return g.seg(tp.rank_idx[o] * (L / tp.dom_size[q]));
  }
  // where a final element at tile offset c goes: y on the root, else the root's fin buffer
  __device__ T* final_dst(size_t tb, size_t c, int slot) const {
    if (me == root) return y + tb + c;
    const int dr = tp.dom_size[tp.rank_dom[root]];
    return slot_ptr<T>(a, root, ch, slot) + s2_off(dr) + (size_t)D * (TL / dr) + c;
  }
  __device__ void stage(int s, size_t t, int slot) {
    const size_t tb = t * TL, len = min(TL, a.count - tb);
    const Geo g{len, TL, L, D};
    const size_t r0 = g.seg(s_lo);
    T* mine = slot_ptr<T>(a, me, ch, slot);
    T* my_s2 = mine + s2_off(d);
    if (s == 0) {  // ---- A: push my data for each domain peer's region ----
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const size_t p0 = g.seg(i * spj), p1 = g.seg((i + 1) * spj);
        cta_copy1<ES>(x + tb + p0, slot_ptr<T>(a, peer(i), ch, slot) + (size_t)cidx(j, i) * Rk, p1 - p0);
      }
    } else if (s == 1) {  // ---- B: domain fold of the other domains' pieces (or of my region if D == 1) ----
      for (int sg = s_lo; sg < s_hi; sg++) {
        for (int q = 0; q < D; q++) {
          if (D > 1 && q == k) continue;
          const size_t c0 = g.piece(sg, q), c1 = g.piece(sg, q + 1);
          if (c1 <= c0) continue;
          PtrList src, dst;
          for (int i = 0; i < d; i++)
            src.add(i == j ? (const void*)(x + tb + c0) : (const void*)(mine + (size_t)cidx(i, j) * Rk + (c0 - r0)));
          if (D == 1) {
            dst.add(final_dst(tb, c0, slot));
          } else {
            const int o = owner_of(tp, q, sg);
            const int dq = tp.dom_size[q];
            dst.add(slot_ptr<T>(a, o, ch, slot) + s2_off(dq) + (size_t)k * (TL / dq) + (c0 - region_lo(g, o)));
          }
          cta_fold<T, OP>(src, dst, c1 - c0);
        }
      }
    } else if (s == 2) {  // ---- C: my pieces: domain fold + cross fold -> the root ----
      for (int sg = s_lo; sg < s_hi; sg++) {
        const size_t c0 = g.piece(sg, k), c1 = g.piece(sg, k + 1);
        if (c1 <= c0) continue;
        PtrList inner, outer, dst;
        for (int i = 0; i < d; i++)
          inner.add(i == j ? (const void*)(x + tb + c0) : (const void*)(mine + (size_t)cidx(i, j) * Rk + (c0 - r0)));
        for (int q = 0; q < D; q++) outer.add(q == k ? nullptr : (const void*)(my_s2 + (size_t)q * Rk + (c0 - r0)));
        dst.add(final_dst(tb, c0, slot));
        cta_fold_hier<T, OP>(inner, k, outer, dst, c1 - c0);
      }
    } else {  // ---- D: the root copies every other rank's final pieces into y ----
      if (me != root) return;
      const T* fin = mine + s2_off(d) + (size_t)D * Rk;
      for (int sg = 0; sg < L; sg++)
        for (int q = 0; q < D; q++) {
          const int o = owner_of(tp, q, sg);
          if (o == root) continue;
          const size_t c0 = D == 1 ? g.seg(sg) : g.piece(sg, q), c1 = D == 1 ? g.seg(sg + 1) : g.piece(sg, q + 1);
          if (c1 > c0) cta_copy1<ES>(fin + c0, y + tb + c0, c1 - c0);
        }
    }
  }
};

// ================================================================== All-to-All (NEXT-2) ========
// out_r[j*B + t] = x_j[r*B + t] (B = count per block). Every block crosses NVLink once, straight to its
// destination's scratch (NVSwitch gives every pair full bandwidth, so there is nothing to aggregate per
// domain). Slot layout: in[n-1][T] (compact sender index). Stages: 0 A push blocks | 1 B copy-out.
template <typename T>
struct A2aOp {
  static constexpr bool kSteal = false;
  static constexpr int ES = sizeof(T);
  const OpArgs& a;
  int me, ch, n;
  size_t TL, Bc;
  const T* x;
  T* y;
  __device__ A2aOp(const OpArgs& a_, int row, int ch_) : a(a_), ch(ch_) {
    me = a.local_rank[row];
    n = a.topo.n;
    TL = a.tile;
    Bc = a.count;
    x = (const T*)a.send[row];
    y = (T*)a.recv[row];
  }
  __device__ void stage(int s, size_t t, int slot) {
    const size_t tb = t * TL, len = min(TL, Bc - tb);
    if (s == 0) {
      for (int r = 0; r < n; r++) {
        if (r == me) cta_copy1<ES>(x + (size_t)me * Bc + tb, y + (size_t)me * Bc + tb, len);
        else cta_copy1<ES>(x + (size_t)r * Bc + tb, slot_ptr<T>(a, r, ch, slot) + (size_t)cidx(me, r) * TL, len);
      }
    } else {
      const T* mine = slot_ptr<T>(a, me, ch, slot);
      for (int r = 0; r < n; r++)
        if (r != me) cta_copy1<ES>(mine + (size_t)cidx(r, me) * TL, y + (size_t)r * Bc + tb, len);
    }
  }
};

// ================================================================== kernels ===================
template <typename T, int OP>
__global__ void __launch_bounds__(kThreads, HETCCL_KERNEL_CPS) k_allreduce(const __grid_constant__ OpArgs a) {
  ArOp<T, OP> op(a, blockIdx.y, blockIdx.x);
  run_pipeline(a, op, op.me, blockIdx.x);
}
template <typename T, int OP>
__global__ void __launch_bounds__(kThreads, HETCCL_KERNEL_CPS) k_reduce_scatter(const __grid_constant__ OpArgs a) {
  RsOp<T, OP> op(a, blockIdx.y, blockIdx.x);
  run_pipeline(a, op, op.me, blockIdx.x);
}
template <typename T>
__global__ void __launch_bounds__(kThreads, HETCCL_KERNEL_CPS) k_all_gather(const __grid_constant__ OpArgs a) {
  AgOp<T> op(a, blockIdx.y, blockIdx.x);
  run_pipeline(a, op, op.me, blockIdx.x);
}
template <typename T, int OP>
__global__ void __launch_bounds__(kThreads, HETCCL_KERNEL_CPS) k_reduce(const __grid_constant__ OpArgs a) {
  RdOp<T, OP> op(a, blockIdx.y, blockIdx.x);
  run_pipeline(a, op, op.me, blockIdx.x);
}
template <typename T>
__global__ void __launch_bounds__(kThreads, HETCCL_KERNEL_CPS) k_all_to_all(const __grid_constant__ OpArgs a) {
  A2aOp<T> op(a, blockIdx.y, blockIdx.x);
  run_pipeline(a, op, op.me, blockIdx.x);
}
template <typename T>
__global__ void __launch_bounds__(kThreads, HETCCL_KERNEL_CPS) k_broadcast(const __grid_constant__ OpArgs a) {
  BcOp<T> op(a, blockIdx.y, blockIdx.x);
  run_pipeline(a, op, op.me, blockIdx.x);
}

// ================================================================== one-shot All-Reduce (NEXT-3) =
// Small messages are latency-bound: the five-stage hierarchy costs five flag round trips. Here every
// rank pushes its whole chunk into every peer's one-shot area (double-buffered by op parity), signals
// once, waits for the n-1 others, and reduces all n operands locally in the oracle's domain-major
// order (cta_fold_domains) — bitwise identical to the hierarchical path, one round trip.
// Counters per (channel, sender): C_OS (data of op g landed), C_OSACK (op g's buffer consumed).
template <typename T, int OP>
__global__ void __launch_bounds__(kThreads, HETCCL_KERNEL_CPS) k_allreduce_oneshot(const __grid_constant__ OpArgs a) {
  constexpr int V = Tr<T>::V;
  const int row = blockIdx.y, ch = blockIdx.x;
  const int me = a.local_rank[row], n = a.topo.n;
  const T* x = (const T*)a.send[row];
  T* y = (T*)a.recv[row];
  uint64_t* F = chan_flags(a, me, ch);
  uint64_t* B = chan_base(a, me, ch);
  __shared__ unsigned long long ops0;
  __shared__ int abort_;
  if (threadIdx.x == 0) {
    ops0 = B[kCounters * kLineWords + 1];
    abort_ = 0;
    g_dbase = 0;
    g_dnth = blockDim.x;
    g_pf = 1;
    g_tma = 0;  // no ring in the one-shot kernel (its movers take the register path)
    g_lgsts = 0;
  }
  __syncthreads();
  const unsigned long long g = ops0;
  const int buf = (int)(g & 1);
  const size_t chunk = (a.count + (size_t)a.nch * V - 1) / ((size_t)a.nch * V) * V;
  const size_t lo = min(a.count, (size_t)ch * chunk), hi = min(a.count, lo + chunk);
  // channel ch's private region of (owner, buffer, sender): its chunk [lo, hi) lands at offset 0
  auto area = [&](int owner, int sender) -> T* {
    return (T*)(a.mem[owner].scratch + a.os_off + ((size_t)buf * n + sender) * a.os_stride + (size_t)ch * a.os_chan);
  };
  auto wait_all = [&](int ctr, uint64_t target) {
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      if (lane < n && lane != me) {
        const uint64_t* w = F + ctr * kLineWords + lane;
        const uint64_t t0 = globaltimer();
        uint32_t spins = 0;
        while (ld_acquire(w, a.gpu_scope) < target) {
          if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > a.timeout_ns) {
            atomicOr(a.err, 1ull + ((unsigned long long)ctr << 8) + ((unsigned long long)lane << 16));
            abort_ = 1;
            break;
          }
        }
      }
    }
    __syncthreads();
  };
  auto signal_all = [&](int ctr) {
    __syncthreads();
    if (threadIdx.x < 32) {
      fence_acq_rel(a.gpu_scope);
      const int lane = threadIdx.x;
      if (lane < n && lane != me) red_add_relaxed(chan_flags(a, lane, ch) + ctr * kLineWords + me, 1, a.gpu_scope);
    }
  };
  // 1. the buffer of op g-2 must be consumed everywhere before it is overwritten
  if (g >= 2) wait_all(C_OSACK, g - 1);
  if (abort_) return;
  // 2. push my chunk to every peer
  {
    PtrList dst;
    for (int r = 0; r < n; r++)
      if (r != me) dst.add(area(r, me));
    cta_copy<sizeof(T)>(x + lo, dst, hi - lo);
  }
  signal_all(C_OS);
  // 3. wait for every peer's chunk, reduce all n operands in the oracle's order
  wait_all(C_OS, g + 1);
  if (abort_) return;
  {
    PtrList src, dst;
    for (int r = 0; r < n; r++) src.add(r == me ? (const void*)(x + lo) : (const void*)area(me, r));
    dst.add(y + lo);
    cta_fold_domains<T, OP>(src, a.topo, dst, hi - lo);
  }
  signal_all(C_OSACK);  // my reads of this buffer are done
  if (threadIdx.x == 0) B[kCounters * kLineWords + 1] = g + 1;
}

// ================================================================== n = 1 (a9) ================
template <int ES>
__global__ void __launch_bounds__(kThreads) k_copy(const void* src, void* dst, size_t n) {
  constexpr int V = 16 / ES;
  const bool al = (((uintptr_t)src | (uintptr_t)dst) & 15) == 0;
  const size_t nv = al ? n / V : 0;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  for (size_t v0 = tid; v0 < nv; v0 += kCopyUnroll * nth) {
    uint4 w[kCopyUnroll];
#pragma unroll
    for (int u = 0; u < kCopyUnroll; u++)
      if (v0 + u * nth < nv) w[u] = ld_v4((const char*)src + (v0 + u * nth) * 16);
#pragma unroll
    for (int u = 0; u < kCopyUnroll; u++)
      if (v0 + u * nth < nv) st_v4((char*)dst + (v0 + u * nth) * 16, w[u]);
  }
  for (size_t i = nv * V + tid; i < n; i += nth) {
    if (ES == 4) st_s32((char*)dst + i * 4, ld_s32((const char*)src + i * 4));
    else st_s16((char*)dst + i * 2, ld_s16((const char*)src + i * 2));
  }
}

// ================================================================== launch ====================
typedef void (*KernFn)(OpArgs);

static KernFn pick_oneshot(int dt, int red) {
#define HC_OS(T)                                                       \
  if (red == RED_SUM) return (KernFn)k_allreduce_oneshot<T, RED_SUM>; \
  if (red == RED_MAX) return (KernFn)k_allreduce_oneshot<T, RED_MAX>; \
  return (KernFn)k_allreduce_oneshot<T, RED_MIN>;
  switch (dt) {
    case DT_F32: { HC_OS(float) }
    case DT_INT32: { HC_OS(int32_t) }
    case DT_BF16: { HC_OS(__nv_bfloat16) }
    case DT_F16: { HC_OS(__half) }
  }
#undef HC_OS
  return nullptr;
}

template <typename T>
static KernFn pick_reduce(int op, int red) {
  if (op == OP_REDUCE) {
    if (red == RED_SUM) return (KernFn)k_reduce<T, RED_SUM>;
    if (red == RED_MAX) return (KernFn)k_reduce<T, RED_MAX>;
    return (KernFn)k_reduce<T, RED_MIN>;
  }
  if (op == OP_ALLREDUCE) {
    if (red == RED_SUM) return (KernFn)k_allreduce<T, RED_SUM>;
    if (red == RED_MAX) return (KernFn)k_allreduce<T, RED_MAX>;
    return (KernFn)k_allreduce<T, RED_MIN>;
  }
  if (red == RED_SUM) return (KernFn)k_reduce_scatter<T, RED_SUM>;
  if (red == RED_MAX) return (KernFn)k_reduce_scatter<T, RED_MAX>;
  return (KernFn)k_reduce_scatter<T, RED_MIN>;
}

static KernFn pick(int op, int dt, int red) {
  if (op == OP_ALLREDUCE || op == OP_REDUCE_SCATTER || op == OP_REDUCE) {
    switch (dt) {
      case DT_F32: return pick_reduce<float>(op, red);
      case DT_INT32: return pick_reduce<int32_t>(op, red);
      case DT_BF16: return pick_reduce<__nv_bfloat16>(op, red);
      case DT_F16: return pick_reduce<__half>(op, red);
    }
    return nullptr;
  }
  const bool two = (dt == DT_BF16 || dt == DT_F16);
  if (op == OP_ALL_GATHER) return two ? (KernFn)k_all_gather<__half> : (KernFn)k_all_gather<float>;
  if (op == OP_BROADCAST) return two ? (KernFn)k_broadcast<__half> : (KernFn)k_broadcast<float>;
  if (op == OP_ALL_TO_ALL) return two ? (KernFn)k_all_to_all<__half> : (KernFn)k_all_to_all<float>;
  return nullptr;
}

// dynamic shared memory of a launch: the TMA ring for the pipeline kernels when the op uses it
static size_t dyn_smem(int op, int tma) {
  if (op == OP_ALLREDUCE_ONESHOT) return 0;
  if (HETCCL_LEGACY_MOVERS) return kStageBytes;  // cp.async staging slots
  return (HETCCL_TMA && tma) ? (size_t)kTmaStages * kTmaStageBytes : 0;
}

// per-process memo of (kernel, device) -> dynamic-smem opt-in done / co-resident CTAs per SM: both are host API
// calls that would otherwise sit on every op's launch path (small-message latency)
struct FnMemo {
  KernFn fn;
  int dev;
  size_t smem;
  int per_sm;  // -1: not queried yet
};
static FnMemo g_memo[512];
static int g_nmemo = 0;
static std::mutex g_memo_mu;
static FnMemo* memo(KernFn fn, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_memo_mu);
  for (int i = 0; i < g_nmemo; i++)
    if (g_memo[i].fn == fn && g_memo[i].dev == dev && g_memo[i].smem == smem) return &g_memo[i];
  if (g_nmemo == 512) return nullptr;
  FnMemo* m = &g_memo[g_nmemo];
  if (smem > 0 &&  // (static + dynamic > 48 KiB needs the opt-in even for 48 KiB dynamic)
      cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return nullptr;
  *m = FnMemo{fn, dev, smem, -1};
  g_nmemo++;
  return m;
}
static cudaError_t allow_smem(KernFn fn, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  return memo(fn, bytes) ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_collective(const OpArgs& a, int nlocal, int dt, int red, bool cooperative, cudaStream_t s) {
  KernFn fn = a.op == OP_ALLREDUCE_ONESHOT ? pick_oneshot(dt, red) : pick(a.op, dt, red);
  if (!fn) return cudaErrorInvalidValue;
  const size_t smem = dyn_smem(a.op, a.tma);
  cudaError_t e = allow_smem(fn, smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.nch, nlocal), block(kThreads);
  void* args[] = {(void*)&a};
  if (cooperative) return cudaLaunchCooperativeKernel((const void*)fn, grid, block, args, smem, s);
  return cudaLaunchKernel((const void*)fn, grid, block, args, smem, s);
}

cudaError_t launch_copy(const void* src, void* dst, size_t n, int es, cudaStream_t s) {
  if (n == 0 || src == dst) return cudaSuccess;
  size_t bytes = n * es;
  int blocks = (int)std::min<size_t>(148 * 2, (bytes + 16 * kThreads * kCopyUnroll - 1) / (16 * kThreads * kCopyUnroll));
  if (blocks < 1) blocks = 1;
  if (es == 4) k_copy<4><<<blocks, kThreads, 0, s>>>(src, dst, n);
  else k_copy<2><<<blocks, kThreads, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

// max co-resident CTAs of a collective kernel on this device (for the cooperative mux launch)
int max_coresident(int op, int dt, int red, int tma) {
  KernFn fn = op == OP_ALLREDUCE_ONESHOT ? pick_oneshot(dt, red) : pick(op, dt, red);
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = dyn_smem(op, tma);
  FnMemo* m = memo(fn, smem);
  if (!m) return 0;
  if (m->per_sm < 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, kThreads, smem) != cudaSuccess) return 0;
    m->per_sm = per_sm;
  }
  return m->per_sm * sms;
}

}  // namespace HETCCL_KNS
}  // namespace hetccl
