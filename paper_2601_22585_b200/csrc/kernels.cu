// kernels.cu — sm_100a device code of the hierarchical collectives.
//
// One persistent CTA per (channel, local rank). A channel walks the tiles t = ch, ch+nch, ... of the
// op; every stage of a tile moves data with 16-byte vector loads/stores — remote stores go straight
// into a peer's IPC-mapped scratch slot over NVLink 5 / NVSwitch ("push"), all reads are local —
// and hands off to the next stage through per-(rank, channel, stage) counters:
//   writer: data stores -> __syncthreads -> fence.acq_rel.sys -> red.relaxed.sys.add(+1) on the
//           receiver's counter;
//   reader: thread 0 spins ld.acquire.sys until the counter reaches its cumulative target ->
//           __syncthreads -> ld.global.cg of the staged data.
// Slots are a ring of kNumSlots per channel; before writing tile t a rank waits until every
// receiver has acked tile t - kNumSlots (C_ACK). Targets are cumulative across launches (bases kept
// in the rank's own flag line C_BASE), so the protocol needs no host sequence numbers and replays
// under CUDA graphs. The same kernels serve the rank-multiplexed mode (all ranks on one device,
// rank = blockIdx.y, cooperative launch) and the one-rank-per-GPU mode (gridDim.y = 1).
//
// Arithmetic (readings R3, R5, R6, R8): per element, fold ascending rank inside a domain
// (seeded with the first operand), narrow 16-bit types once at the domain boundary (stored partial),
// fold the D partials in ascending domain id, narrow once more. fp32 accumulation for bf16/fp16,
// IEEE RNE everywhere (__fadd_rn, __float2bfloat16_rn, __float2half_rn), uint32 wrap for int32.
// Built without --use_fast_math (no FTZ, reading R9).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "hetccl_internal.h"

namespace hetccl {

// ------------------------------------------------------------------ PTX primitives -------------
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void red_add_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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
  __device__ PtrList() : n(0) {}
  __device__ void add(const void* q) { p[n++] = q; }
};

__device__ __forceinline__ bool all_aligned16(const PtrList& a, const PtrList& b) {
  uintptr_t o = 0;
  for (int i = 0; i < a.n; i++) o |= (uintptr_t)a.p[i];
  for (int i = 0; i < b.n; i++) o |= (uintptr_t)b.p[i];
  return (o & 15) == 0;
}

constexpr int kUnroll = 4;

// dst[d][i] = src[i] for every destination d, i < n elements of size ES (bit copy)
template <int ES>
__device__ void cta_copy(const void* src, const PtrList& dsts, size_t n) {
  if (n == 0) return;
  constexpr int V = 16 / ES;
  const int tid = threadIdx.x, nth = blockDim.x;
  PtrList s1;
  s1.add(src);
  const size_t nv = all_aligned16(s1, dsts) ? n / V : 0;
  const char* sp = (const char*)src;
  for (size_t v0 = tid; v0 < nv; v0 += (size_t)kUnroll * nth) {
    uint4 w[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; u++) {
      size_t v = v0 + (size_t)u * nth;
      if (v < nv) w[u] = ld_v4(sp + v * 16);
    }
    for (int d = 0; d < dsts.n; d++) {
      char* dp = (char*)dsts.p[d];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
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
__device__ void cta_fold(const PtrList& srcs, const PtrList& dsts, size_t n) {
  using TR = Tr<T>;
  using S = typename TR::S;
  using A = typename TR::A;
  constexpr int V = TR::V;
  if (n == 0) return;
  if (srcs.n == 1) {  // a single operand: the value is already in the dtype (bit copy)
    cta_copy<sizeof(S)>(srcs.p[0], dsts, n);
    return;
  }
  const int tid = threadIdx.x, nth = blockDim.x;
  const size_t nv = all_aligned16(srcs, dsts) ? n / V : 0;
  for (size_t v0 = tid; v0 < nv; v0 += (size_t)kUnroll * nth) {
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

// ------------------------------------------------------------------ protocol helpers -----------
__device__ __forceinline__ uint64_t* chan_flags(const OpArgs& a, int rank, int ch) {
  return a.mem[rank].flags + (size_t)ch * kChanWords;
}

template <typename T>
__device__ __forceinline__ T* slot_ptr(const OpArgs& a, int rank, int ch, int slot) {
  return (T*)(a.mem[rank].scratch + ((size_t)(ch * kNumSlots + slot) * a.slot_elems) * sizeof(T));
}

struct CtaState {
  unsigned long long base[C_NREMOTE];
  int abort_;
};

__device__ __forceinline__ void cta_begin(CtaState& st, const uint64_t* F) {
  if (threadIdx.x == 0) {
    for (int c = 0; c < C_NREMOTE; c++) st.base[c] = F[C_BASE * kFlagStride + c];
    st.abort_ = 0;
  }
  __syncthreads();
}

// all threads: completes every data store of this CTA, then adds cnt[r] to counter `ctr` of
// channel `ch` on every rank r with cnt[r] > 0 (lane r of warp 0 signals rank r)
__device__ __forceinline__ void cta_signal(const OpArgs& a, int ch, int ctr, const uint32_t* cnt) {
  __syncthreads();
  if (threadIdx.x < 32) {
    fence_acq_rel_sys();
    const int r = threadIdx.x;
    if (r < a.topo.n && cnt[r]) red_add_relaxed_sys(chan_flags(a, r, ch) + ctr * kFlagStride, cnt[r]);
  }
}

__device__ __forceinline__ void cta_signal_mask(const OpArgs& a, int ch, int ctr, uint32_t mask) {
  __syncthreads();
  if (threadIdx.x < 32) {
    fence_acq_rel_sys();
    const int r = threadIdx.x;
    if ((mask >> r) & 1u) red_add_relaxed_sys(chan_flags(a, r, ch) + ctr * kFlagStride, 1);
  }
}

// all threads: wait until my counter `ctr` >= target (thread 0 polls); false on timeout
__device__ __noinline__ bool cta_wait(const OpArgs& a, CtaState& st, const uint64_t* F, int ctr, uint64_t target) {
  if (threadIdx.x == 0) {
    const uint64_t* p = F + ctr * kFlagStride;
    if (ld_acquire_sys(p) < target) {
      const uint64_t t0 = globaltimer();
      uint32_t it = 0;
      while (ld_acquire_sys(p) < target) {
        if ((++it & 1023u) == 0 && (long long)(globaltimer() - t0) > a.timeout_ns) {
          atomicOr(a.err, 1ull + ((unsigned long long)ctr << 8));
          *(volatile int*)&st.abort_ = 1;
          break;
        }
      }
    }
  }
  __syncthreads();
  return *(volatile int*)&st.abort_ == 0;
}

__device__ __forceinline__ void cta_end(CtaState& st, uint64_t* F, const RankPlan& rp, int tiles_done) {
  __syncthreads();
  if (threadIdx.x == 0 && st.abort_ == 0)
    for (int c = 0; c < C_NREMOTE; c++) F[C_BASE * kFlagStride + c] = st.base[c] + (uint64_t)tiles_done * rp.inc[c];
}

__device__ __forceinline__ uint64_t ack_target(const CtaState& st, const RankPlan& rp, int tl) {
  return st.base[C_ACK] + (uint64_t)(tl >= kNumSlots ? tl - kNumSlots + 1 : 0) * rp.inc[C_ACK];
}

__device__ __forceinline__ size_t floor_to(size_t x, size_t q) { return x / q * q; }

// elementary-segment and piece boundaries of one tile (same formulas as plan.cpp)
struct Geo {
  size_t len;
  int L, D, V;
  __device__ size_t seg(int s) const { return s >= L ? len : floor_to(len * (size_t)s / L, V); }
  __device__ size_t piece(int s, int p) const {
    size_t b0 = seg(s), b1 = seg(s + 1);
    return p >= D ? b1 : b0 + floor_to((b1 - b0) * (size_t)p / D, V);
  }
};

// piece i of dd of a shard tile of length len (RS / AG)
__device__ __forceinline__ size_t sub_lo(size_t len, int dd, int i, int V) {
  return i >= dd ? len : floor_to(len * (size_t)i / dd, V);
}

__device__ __forceinline__ int owner_of(const Topo& t, int q, int s) {
  return t.members[t.dom_first[q] + s / (t.L / t.dom_size[q])];
}

// ================================================================== All-Reduce (a1-a5) =========
// Slot layout on a rank of domain k (d = d_k, Rk = tile/d):
//   s1[d][Rk] | s2[D][Rk] | ag[Rk] | s3[d][Rk]
template <typename T, int OP>
__global__ void __launch_bounds__(kThreads, 1) k_allreduce(const __grid_constant__ OpArgs a) {
  constexpr int ES = sizeof(T);
  constexpr int V = Tr<T>::V;
  __shared__ CtaState st;
  const int row = blockIdx.y, ch = blockIdx.x;
  const int me = a.local_rank[row];
  const Topo& tp = a.topo;
  const int k = tp.rank_dom[me], j = tp.rank_idx[me], d = tp.dom_size[k], D = tp.D, L = tp.L;
  const int spj = L / d, s_lo = j * spj, s_hi = s_lo + spj;
  const size_t TL = a.tile, Rk = TL / d;
  const T* x = (const T*)a.send[row];
  T* y = (T*)a.recv[row];
  uint64_t* F = chan_flags(a, me, ch);
  const RankPlan& rp = a.rp[me];
  uint32_t dpeers = 0;
  for (int i = 0; i < d; i++)
    if (i != j) dpeers |= 1u << tp.members[tp.dom_first[k] + i];
  cta_begin(st, F);
  int tl = 0;
  for (size_t t = ch; t < a.ntiles; t += a.nch, ++tl) {
    const size_t tb = t * TL, len = min(TL, a.count - tb);
    const Geo g{len, L, D, V};
    const int slot = tl % kNumSlots;
    if (!cta_wait(a, st, F, C_ACK, ack_target(st, rp, tl))) break;
    const size_t r0 = g.seg(s_lo), r1 = g.seg(s_hi);
    T* mine = slot_ptr<T>(a, me, ch, slot);
    T* my_ag = mine + TL + (size_t)D * Rk;
    // ---- a1: intra-domain reduce-scatter, push my slices to their owners' s1[j] ----
    if (d > 1) {
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const int peer = tp.members[tp.dom_first[k] + i];
        const size_t p0 = g.seg(i * spj), p1 = g.seg((i + 1) * spj);
        cta_copy1<ES>(x + tb + p0, slot_ptr<T>(a, peer, ch, slot) + (size_t)j * Rk, p1 - p0);
      }
      cta_signal_mask(a, ch, C_S1, dpeers);
      if (!cta_wait(a, st, F, C_S1, st.base[C_S1] + (uint64_t)(tl + 1) * rp.inc[C_S1])) break;
    }
    // ---- fold my region over the domain (ascending rank); route each piece to its reducer ----
    for (int s = s_lo; s < s_hi; s++) {
      for (int q = 0; q < D; q++) {
        const size_t c0 = g.piece(s, q), c1 = g.piece(s, q + 1);
        if (c1 <= c0) continue;
        PtrList src, dst;
        for (int i = 0; i < d; i++)
          src.add(i == j ? (const void*)(x + tb + c0) : (const void*)(mine + (size_t)i * Rk + (c0 - r0)));
        if (D == 1) {
          dst.add(y + tb + c0);
          if (d > 1) dst.add(my_ag + (c0 - r0));
        } else if (q == k) {
          dst.add(mine + TL + (size_t)k * Rk + (c0 - r0));
        } else {
          const int o = owner_of(tp, q, s);
          const int dq = tp.dom_size[q];
          const size_t ro = g.seg(tp.rank_idx[o] * (L / dq));
          dst.add(slot_ptr<T>(a, o, ch, slot) + TL + (size_t)k * (TL / dq) + (c0 - ro));
        }
        cta_fold<T, OP>(src, dst, c1 - c0);
      }
    }
    // ---- a2: cross-domain reduce-scatter + all-gather of the partials among segment owners ----
    if (D > 1) {
      __shared__ uint32_t cnt[kMaxRanks];
      if (threadIdx.x < kMaxRanks) {
        int c = 0;
        for (int s = s_lo; s < s_hi; s++)
          for (int q = 0; q < D; q++)
            if (q != k && owner_of(tp, q, s) == (int)threadIdx.x) c++;
        cnt[threadIdx.x] = (uint32_t)c;
      }
      cta_signal(a, ch, C_S2, cnt);
      if (!cta_wait(a, st, F, C_S2, st.base[C_S2] + (uint64_t)(tl + 1) * rp.inc[C_S2])) break;
      for (int s = s_lo; s < s_hi; s++) {
        const size_t c0 = g.piece(s, k), c1 = g.piece(s, k + 1);
        if (c1 <= c0) continue;
        PtrList src, dst;
        for (int q = 0; q < D; q++) src.add(mine + TL + (size_t)q * Rk + (c0 - r0));
        dst.add(y + tb + c0);
        dst.add(my_ag + (c0 - r0));
        for (int q = 0; q < D; q++) {
          if (q == k) continue;
          const int o = owner_of(tp, q, s);
          const int dq = tp.dom_size[q];
          const size_t ro = g.seg(tp.rank_idx[o] * (L / dq));
          dst.add(slot_ptr<T>(a, o, ch, slot) + TL + (size_t)D * (TL / dq) + (c0 - ro));
        }
        cta_fold<T, OP>(src, dst, c1 - c0);
      }
      cta_signal(a, ch, C_AG, cnt);
      if (!cta_wait(a, st, F, C_AG, st.base[C_AG] + (uint64_t)(tl + 1) * rp.inc[C_AG])) break;
    }
    // ---- a3: intra-domain all-gather of the final region ----
    if (d > 1) {
      PtrList dst;
      if (D > 1) dst.add(y + tb + r0);
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const int peer = tp.members[tp.dom_first[k] + i];
        dst.add(slot_ptr<T>(a, peer, ch, slot) + TL + (size_t)(D + 1) * Rk + (size_t)j * Rk);
      }
      cta_copy<ES>(my_ag, dst, r1 - r0);
      cta_signal_mask(a, ch, C_S3, dpeers);
      if (!cta_wait(a, st, F, C_S3, st.base[C_S3] + (uint64_t)(tl + 1) * rp.inc[C_S3])) break;
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const size_t p0 = g.seg(i * spj), p1 = g.seg((i + 1) * spj);
        cta_copy1<ES>(mine + TL + (size_t)(D + 1) * Rk + (size_t)i * Rk, y + tb + p0, p1 - p0);
      }
    } else if (D > 1) {
      cta_copy1<ES>(my_ag, y + tb + r0, r1 - r0);
    }
    // ---- tile done: every slot my senders wrote is consumed ----
    cta_signal_mask(a, ch, C_ACK, rp.partners);
  }
  cta_end(st, F, rp, tl);
}

// ================================================================== Reduce-Scatter (a6) ========
// Per tile (per-shard offsets [tb, tb+len)), member j of domain k owns: its own shard, plus piece j
// (of d) of every other-domain shard. Slot layout on a rank of domain k (RG = T + (n-d)*T/d):
//   s1[d][RG] | s2[D][T]    (s1 region: own-shard part at 0, other-domain shard ro at T + ro*T/d)
template <typename T, int OP>
__global__ void __launch_bounds__(kThreads, 1) k_reduce_scatter(const __grid_constant__ OpArgs a) {
  constexpr int ES = sizeof(T);
  constexpr int V = Tr<T>::V;
  __shared__ CtaState st;
  const int row = blockIdx.y, ch = blockIdx.x;
  const int me = a.local_rank[row];
  const Topo& tp = a.topo;
  const int n = tp.n, k = tp.rank_dom[me], j = tp.rank_idx[me], d = tp.dom_size[k], D = tp.D;
  const size_t TL = a.tile, R = a.count, Pc = TL / d, RG = TL + (size_t)(n - d) * Pc;
  const T* x = (const T*)a.send[row];
  T* y = (T*)a.recv[row];
  uint64_t* F = chan_flags(a, me, ch);
  const RankPlan& rp = a.rp[me];
  uint32_t dpeers = 0, others = 0;
  for (int r = 0; r < n; r++) {
    if (r == me) continue;
    if (tp.rank_dom[r] == k) dpeers |= 1u << r;
    else others |= 1u << r;
  }
  cta_begin(st, F);
  int tl = 0;
  for (size_t t = ch; t < a.ntiles; t += a.nch, ++tl) {
    const size_t tb = t * TL, len = min(TL, R - tb);
    const int slot = tl % kNumSlots;
    if (!cta_wait(a, st, F, C_ACK, ack_target(st, rp, tl))) break;
    T* mine = slot_ptr<T>(a, me, ch, slot);
    const size_t pj0 = sub_lo(len, d, j, V), pj1 = sub_lo(len, d, j + 1, V);
    // ---- intra-domain reduce-scatter: send each peer the data of its region ----
    if (d > 1) {
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const int peer = tp.members[tp.dom_first[k] + i];
        T* dst = slot_ptr<T>(a, peer, ch, slot) + (size_t)j * RG;
        cta_copy1<ES>(x + (size_t)peer * R + tb, dst, len);
        const size_t pi0 = sub_lo(len, d, i, V), pi1 = sub_lo(len, d, i + 1, V);
        int ro = 0;
        for (int r = 0; r < n; r++) {
          if (tp.rank_dom[r] == k) continue;
          cta_copy1<ES>(x + (size_t)r * R + tb + pi0, dst + TL + (size_t)ro * Pc, pi1 - pi0);
          ro++;
        }
      }
      cta_signal_mask(a, ch, C_S1, dpeers);
      if (!cta_wait(a, st, F, C_S1, st.base[C_S1] + (uint64_t)(tl + 1) * rp.inc[C_S1])) break;
    }
    // ---- fold: own shard -> my domain partial; my pieces of other shards -> their owners' s2[k] ----
    {
      PtrList src, dst;
      for (int i = 0; i < d; i++)
        src.add(i == j ? (const void*)(x + (size_t)me * R + tb) : (const void*)(mine + (size_t)i * RG));
      if (D == 1) dst.add(y + tb);
      else dst.add(mine + (size_t)d * RG + (size_t)k * TL);
      cta_fold<T, OP>(src, dst, len);
    }
    if (D > 1) {
      int ro = 0;
      for (int r = 0; r < n; r++) {
        if (tp.rank_dom[r] == k) continue;
        PtrList src, dst;
        for (int i = 0; i < d; i++)
          src.add(i == j ? (const void*)(x + (size_t)r * R + tb + pj0)
                         : (const void*)(mine + (size_t)i * RG + TL + (size_t)ro * Pc));
        const int dr = tp.dom_size[tp.rank_dom[r]];
        const size_t RGr = TL + (size_t)(n - dr) * (TL / dr);
        dst.add(slot_ptr<T>(a, r, ch, slot) + (size_t)dr * RGr + (size_t)k * TL + pj0);
        cta_fold<T, OP>(src, dst, pj1 - pj0);
        ro++;
      }
      cta_signal_mask(a, ch, C_S2, others);
      // ---- cross-domain: fold the D domain partials of my shard (ascending domain id) ----
      if (!cta_wait(a, st, F, C_S2, st.base[C_S2] + (uint64_t)(tl + 1) * rp.inc[C_S2])) break;
      PtrList src, dst;
      for (int q = 0; q < D; q++) src.add(mine + (size_t)d * RG + (size_t)q * TL);
      dst.add(y + tb);
      cta_fold<T, OP>(src, dst, len);
    }
    cta_signal_mask(a, ch, C_ACK, rp.partners);
  }
  cta_end(st, F, rp, tl);
}

// ================================================================== All-Gather (a7) ============
// Mirror of reduce-scatter. Slot layout on a rank of domain k (RG = T + (n-d)*T/d):
//   s_in[d][RG] | xin[n-d][T/d]
template <typename T>
__global__ void __launch_bounds__(kThreads, 1) k_all_gather(const __grid_constant__ OpArgs a) {
  constexpr int ES = sizeof(T);
  constexpr int V = Tr<T>::V;
  __shared__ CtaState st;
  const int row = blockIdx.y, ch = blockIdx.x;
  const int me = a.local_rank[row];
  const Topo& tp = a.topo;
  const int n = tp.n, k = tp.rank_dom[me], j = tp.rank_idx[me], d = tp.dom_size[k], D = tp.D;
  const size_t TL = a.tile, R = a.count, Pc = TL / d, RG = TL + (size_t)(n - d) * Pc;
  const T* x = (const T*)a.send[row];
  T* y = (T*)a.recv[row];
  uint64_t* F = chan_flags(a, me, ch);
  const RankPlan& rp = a.rp[me];
  uint32_t dpeers = 0, others = 0;
  for (int r = 0; r < n; r++) {
    if (r == me) continue;
    if (tp.rank_dom[r] == k) dpeers |= 1u << r;
    else others |= 1u << r;
  }
  const bool inplace = (x == y + (size_t)me * R);
  cta_begin(st, F);
  int tl = 0;
  for (size_t t = ch; t < a.ntiles; t += a.nch, ++tl) {
    const size_t tb = t * TL, len = min(TL, R - tb);
    const int slot = tl % kNumSlots;
    if (!cta_wait(a, st, F, C_ACK, ack_target(st, rp, tl))) break;
    T* mine = slot_ptr<T>(a, me, ch, slot);
    T* xin = mine + (size_t)d * RG;
    const size_t pj0 = sub_lo(len, d, j, V), pj1 = sub_lo(len, d, j + 1, V);
    if (!inplace) cta_copy1<ES>(x + tb, y + (size_t)me * R + tb, len);
    // ---- cross-domain: piece i of my shard to member i of every other domain ----
    if (D > 1) {
      for (int r = 0; r < n; r++) {
        const int q = tp.rank_dom[r];
        if (q == k) continue;
        const int dq = tp.dom_size[q], i = tp.rank_idx[r];
        int ro_me = 0;  // my index among the ranks outside domain q
        for (int r2 = 0; r2 < me; r2++)
          if (tp.rank_dom[r2] != q) ro_me++;
        const size_t a0 = sub_lo(len, dq, i, V), a1 = sub_lo(len, dq, i + 1, V);
        const size_t RGq = TL + (size_t)(n - dq) * (TL / dq);
        cta_copy1<ES>(x + tb + a0, slot_ptr<T>(a, r, ch, slot) + (size_t)dq * RGq + (size_t)ro_me * (TL / dq), a1 - a0);
      }
      cta_signal_mask(a, ch, C_S2, others);
      if (!cta_wait(a, st, F, C_S2, st.base[C_S2] + (uint64_t)(tl + 1) * rp.inc[C_S2])) break;
    }
    // ---- intra-domain: my region (own shard + received pieces) to every domain peer ----
    {
      PtrList dst_shard;
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const int peer = tp.members[tp.dom_first[k] + i];
        dst_shard.add(slot_ptr<T>(a, peer, ch, slot) + (size_t)j * RG);
      }
      if (dst_shard.n) cta_copy<ES>(x + tb, dst_shard, len);
      int ro = 0;
      for (int r = 0; r < n; r++) {
        if (tp.rank_dom[r] == k) continue;
        PtrList dst;
        dst.add(y + (size_t)r * R + tb + pj0);
        for (int i = 0; i < d; i++) {
          if (i == j) continue;
          const int peer = tp.members[tp.dom_first[k] + i];
          dst.add(slot_ptr<T>(a, peer, ch, slot) + (size_t)j * RG + TL + (size_t)ro * Pc);
        }
        cta_copy<ES>(xin + (size_t)ro * Pc, dst, pj1 - pj0);
        ro++;
      }
    }
    if (d > 1) {
      cta_signal_mask(a, ch, C_S1, dpeers);
      if (!cta_wait(a, st, F, C_S1, st.base[C_S1] + (uint64_t)(tl + 1) * rp.inc[C_S1])) break;
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const int peer = tp.members[tp.dom_first[k] + i];
        const T* reg = mine + (size_t)i * RG;
        cta_copy1<ES>(reg, y + (size_t)peer * R + tb, len);
        const size_t pi0 = sub_lo(len, d, i, V), pi1 = sub_lo(len, d, i + 1, V);
        int ro = 0;
        for (int r = 0; r < n; r++) {
          if (tp.rank_dom[r] == k) continue;
          cta_copy1<ES>(reg + TL + (size_t)ro * Pc, y + (size_t)r * R + tb + pi0, pi1 - pi0);
          ro++;
        }
      }
    }
    cta_signal_mask(a, ch, C_ACK, rp.partners);
  }
  cta_end(st, F, rp, tl);
}

// ================================================================== Broadcast (a8) =============
// Root -> its domain members (scatter of regions) -> one owner per other domain per segment ->
// intra-domain all-gather. Slot layout on a rank of domain k (Rk = T/d): reg[Rk] | s3[d][Rk]
template <typename T>
__global__ void __launch_bounds__(kThreads, 1) k_broadcast(const __grid_constant__ OpArgs a) {
  constexpr int ES = sizeof(T);
  constexpr int V = Tr<T>::V;
  __shared__ CtaState st;
  const int row = blockIdx.y, ch = blockIdx.x;
  const int me = a.local_rank[row];
  const Topo& tp = a.topo;
  const int k = tp.rank_dom[me], j = tp.rank_idx[me], d = tp.dom_size[k], D = tp.D, L = tp.L;
  const int root = a.root, kr = tp.rank_dom[root];
  const int spj = L / d, s_lo = j * spj, s_hi = s_lo + spj;
  const size_t TL = a.tile, Rk = TL / d;
  const T* x = (const T*)a.send[row];
  T* y = (T*)a.recv[row];
  uint64_t* F = chan_flags(a, me, ch);
  const RankPlan& rp = a.rp[me];
  uint32_t dpeers = 0;
  for (int i = 0; i < d; i++)
    if (i != j) dpeers |= 1u << tp.members[tp.dom_first[k] + i];
  const bool is_root = (me == root);
  cta_begin(st, F);
  int tl = 0;
  for (size_t t = ch; t < a.ntiles; t += a.nch, ++tl) {
    const size_t tb = t * TL, len = min(TL, a.count - tb);
    const Geo g{len, L, 1, V};
    const int slot = tl % kNumSlots;
    if (!cta_wait(a, st, F, C_ACK, ack_target(st, rp, tl))) break;
    T* mine = slot_ptr<T>(a, me, ch, slot);
    const size_t r0 = g.seg(s_lo), r1 = g.seg(s_hi);
    // ---- root scatters the regions of its domain ----
    if (is_root && d > 1) {
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const int peer = tp.members[tp.dom_first[k] + i];
        const size_t p0 = g.seg(i * spj), p1 = g.seg((i + 1) * spj);
        cta_copy1<ES>(x + tb + p0, slot_ptr<T>(a, peer, ch, slot), p1 - p0);
      }
      cta_signal_mask(a, ch, C_S1, dpeers);
    }
    if (k == kr && !is_root) {
      if (!cta_wait(a, st, F, C_S1, st.base[C_S1] + (uint64_t)(tl + 1) * rp.inc[C_S1])) break;
    }
    const T* myreg = is_root ? (x + tb + r0) : mine;
    // ---- cross-domain: root-domain owners send each segment to its owner in every other domain ----
    if (D > 1) {
      if (k == kr) {
        __shared__ uint32_t cnt[kMaxRanks];
        if (threadIdx.x < kMaxRanks) cnt[threadIdx.x] = 0;
        __syncthreads();
        for (int s = s_lo; s < s_hi; s++) {
          const size_t c0 = g.seg(s), c1 = g.seg(s + 1);
          PtrList dst;
          for (int q = 0; q < D; q++) {
            if (q == kr) continue;
            const int o = owner_of(tp, q, s);
            const size_t ro = g.seg(tp.rank_idx[o] * (L / tp.dom_size[q]));
            dst.add(slot_ptr<T>(a, o, ch, slot) + (c0 - ro));
            if (threadIdx.x == 0) cnt[o]++;
          }
          cta_copy<ES>(myreg + (c0 - r0), dst, c1 - c0);
        }
        cta_signal(a, ch, C_S2, cnt);
      } else {
        if (!cta_wait(a, st, F, C_S2, st.base[C_S2] + (uint64_t)(tl + 1) * rp.inc[C_S2])) break;
      }
    }
    // ---- intra-domain all-gather of the regions (nobody sends to the root) ----
    {
      PtrList dst;
      if (!is_root) dst.add(y + tb + r0);
      for (int i = 0; i < d; i++) {
        if (i == j) continue;
        const int peer = tp.members[tp.dom_first[k] + i];
        if (peer == root) continue;
        dst.add(slot_ptr<T>(a, peer, ch, slot) + Rk + (size_t)j * Rk);
      }
      if (dst.n) cta_copy<ES>(myreg, dst, r1 - r0);
      if (is_root && x != y) cta_copy1<ES>(x + tb, y + tb, len);
    }
    if (d > 1) {
      cta_signal_mask(a, ch, C_S3, dpeers & ~(1u << root));
      if (!is_root) {
        if (!cta_wait(a, st, F, C_S3, st.base[C_S3] + (uint64_t)(tl + 1) * rp.inc[C_S3])) break;
        for (int i = 0; i < d; i++) {
          if (i == j) continue;
          const size_t p0 = g.seg(i * spj), p1 = g.seg((i + 1) * spj);
          cta_copy1<ES>(mine + Rk + (size_t)i * Rk, y + tb + p0, p1 - p0);
        }
      }
    }
    cta_signal_mask(a, ch, C_ACK, rp.partners);
  }
  cta_end(st, F, rp, tl);
}

// ================================================================== n = 1 (a9) ================
template <int ES>
__global__ void __launch_bounds__(kThreads) k_copy(const void* src, void* dst, size_t n) {
  constexpr int V = 16 / ES;
  const bool al = (((uintptr_t)src | (uintptr_t)dst) & 15) == 0;
  const size_t nv = al ? n / V : 0;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  for (size_t v0 = tid; v0 < nv; v0 += kUnroll * nth) {
    uint4 w[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
      if (v0 + u * nth < nv) w[u] = ld_v4((const char*)src + (v0 + u * nth) * 16);
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
      if (v0 + u * nth < nv) st_v4((char*)dst + (v0 + u * nth) * 16, w[u]);
  }
  for (size_t i = nv * V + tid; i < n; i += nth) {
    if (ES == 4) st_s32((char*)dst + i * 4, ld_s32((const char*)src + i * 4));
    else st_s16((char*)dst + i * 2, ld_s16((const char*)src + i * 2));
  }
}

// ================================================================== launch ====================
typedef void (*KernFn)(OpArgs);

template <typename T>
static KernFn pick_reduce(int op, int red) {
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
  if (op == OP_ALLREDUCE || op == OP_REDUCE_SCATTER) {
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
  return nullptr;
}

cudaError_t launch_collective(const OpArgs& a, int nlocal, int dt, int red, bool cooperative, cudaStream_t s) {
  KernFn fn = pick(a.op, dt, red);
  if (!fn) return cudaErrorInvalidValue;
  dim3 grid(a.nch, nlocal), block(kThreads);
  if (cooperative) {
    void* args[] = {(void*)&a};
    return cudaLaunchCooperativeKernel((const void*)fn, grid, block, args, 0, s);
  }
  void* args[] = {(void*)&a};
  return cudaLaunchKernel((const void*)fn, grid, block, args, 0, s);
}

cudaError_t launch_copy(const void* src, void* dst, size_t n, int es, cudaStream_t s) {
  if (n == 0 || src == dst) return cudaSuccess;
  size_t bytes = n * es;
  int blocks = (int)std::min<size_t>(148 * 4, (bytes + 16 * kThreads * kUnroll - 1) / (16 * kThreads * kUnroll));
  if (blocks < 1) blocks = 1;
  if (es == 4) k_copy<4><<<blocks, kThreads, 0, s>>>(src, dst, n);
  else k_copy<2><<<blocks, kThreads, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

// max co-resident CTAs of a collective kernel on this device (for the cooperative mux launch)
int max_coresident(int op, int dt, int red) {
  KernFn fn = pick(op, dt, red);
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, kThreads, 0) != cudaSuccess) return 0;
  return per_sm * sms;
}

}  // namespace hetccl
