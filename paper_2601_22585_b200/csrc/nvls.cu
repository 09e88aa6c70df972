// nvls.cu — opt-in NVLink SHARP (NVLS) All-Reduce for single-process multi-GPU communicators
// (HETCCL_NVLS=1 at hetccl_comm_init_all).
//
// The intra-domain stages of the hierarchy run inside the NVSwitch: every domain (all domains of equal
// size d >= 2) gets one multicast object; each member binds a buffer of its own HBM to it ("uc", its
// unicast view) and maps the multicast address ("mc"). Per chunk of CE elements per rank:
//   1. copy x -> uc (zero-padded to a 16-byte vector), signal N_IN to the domain members;
//   2. member i waits for N_IN, reads its segment i through mc with multimem.ld_reduce (the switch
//      sums the d members' copies, fp32 accumulation for bf16/fp16) = this domain's partial P_k,
//      stores it into its own cross slot and pushes it to member i of every other domain (N_X);
//   3. waits for the other domains' partials, folds the D partials in ascending domain id in fp32,
//      narrows once, and multimem.st's the result into every member's uc (one store, the switch
//      replicates), ACKs the cross slots (N_XACK) and signals N_OUT;
//   4. after N_OUT from every member, copies uc -> y.
// 16-bit dtypes are staged in fp32 (HETCCL_NVLS_WIDE=1, default): step 1 widens x into an fp32 uc, the
// switch adds fp32 (round-to-nearest-even on every add, q33/q34 probe; its native 16-bit adds are not RNE)
// and the partial is narrowed once (reading R6) — the same error bound as the oracle's fold, so R7's
// elementwise 1e-2 gate holds — at twice the multicast bytes; the final value goes back through uc in fp32
// (exact) and is narrowed on the way out. When send == recv == the uc buffer itself (hetccl_comm_nvls; f32,
// or 16-bit with HETCCL_NVLS_WIDE=0), steps 1 and 4 are skipped (zero copy).
// The switch's summation order inside a domain is not reading R3's ascending rank order, so this mode
// is tolerance-only (R7 gate; R21), not bit-exact; the cross-domain fold keeps R3's order.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <errno.h>
#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "hetccl_internal.h"

namespace hetccl {

namespace {

constexpr int kNvThreads = 256;
constexpr int kNvCounters = 5;  // N_IN, N_X, N_XACK, N_OUT, N_DONE
enum : int { N_IN = 0, N_X = 1, N_XACK = 2, N_OUT = 3, N_DONE = 4 };
constexpr int kNvSlots = 4;     // chunk slots of the uc buffer and of the cross slots (the pipeline is 4 deep)
constexpr int kNvUnroll = 4;    // multicast reductions in flight per thread

// ---------------------------------------------------------------- device -----------------------
__device__ __forceinline__ uint64_t nv_ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void nv_fence() {
  asm volatile("fence.proxy.alias;" ::: "memory");  // uc and mc are two virtual aliases of one buffer
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ void nv_red(uint64_t* p) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ uint4 nv_ld(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void nv_st(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

template <int DT>
__device__ __forceinline__ uint4 mc_ld_reduce(const void* p);
template <>
__device__ __forceinline__ uint4 mc_ld_reduce<DT_BF16>(const void* p) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
template <>
__device__ __forceinline__ uint4 mc_ld_reduce<DT_F16>(const void* p) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
template <>
__device__ __forceinline__ uint4 mc_ld_reduce<DT_F32>(const void* p) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mc_st(void* p, const uint4& v) {  // bit pattern of 16 bytes
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w) : "memory");
}

// fp32 views of a 16-byte vector
template <int DT>
struct NvVec;
template <>
struct NvVec<DT_BF16> {
  static constexpr int V = 8;
  __device__ static float get(const uint4& w, int e) {
    const uint32_t u = (&w.x)[e >> 1];
    return __uint_as_float((e & 1) ? (u & 0xffff0000u) : (u << 16));
  }
  __device__ static void set(uint4& w, int e, float a) {
    uint32_t& u = (&w.x)[e >> 1];
    const uint32_t s = __bfloat16_as_ushort(__float2bfloat16_rn(a));
    u = (e & 1) ? ((u & 0xffffu) | (s << 16)) : ((u & 0xffff0000u) | s);
  }
};
template <>
struct NvVec<DT_F16> {
  static constexpr int V = 8;
  __device__ static float get(const uint4& w, int e) {
    const uint32_t u = (&w.x)[e >> 1];
    return __half2float(__ushort_as_half((unsigned short)((e & 1) ? (u >> 16) : (u & 0xffffu))));
  }
  __device__ static void set(uint4& w, int e, float a) {
    uint32_t& u = (&w.x)[e >> 1];
    const uint32_t s = __half_as_ushort(__float2half_rn(a));
    u = (e & 1) ? ((u & 0xffffu) | (s << 16)) : ((u & 0xffff0000u) | s);
  }
};
template <>
struct NvVec<DT_F32> {
  static constexpr int V = 4;
  __device__ static float get(const uint4& w, int e) { return __uint_as_float((&w.x)[e]); }
  __device__ static void set(uint4& w, int e, float a) { (&w.x)[e] = __float_as_uint(a); }
};

struct NvlsArgs {
  const char* send;
  char* recv;
  size_t count;       // elements per rank
  size_t ce;          // chunk elements per rank (multiple of d * V)
  char* uc;           // my unicast view of the domain's multicast buffer
  char* mc;           // the domain's multicast address (as mapped on my device)
  char* xs[kMaxRanks];        // cross slots of member i of domain q (q == k: mine)
  uint64_t* fl[kMaxRanks];    // flag area of every rank
  size_t xs_slot;     // bytes of one (slot, sender domain) cross buffer = ce / d elements
  int me, d, D, i, k, nch, zero_copy, wide;
  int dmem[kMaxRanks];        // ranks of my domain, by index
  int xrank[kMaxRanks];       // rank of member i of domain q
  unsigned long long* err;
  long long timeout_ns;
};

__device__ __forceinline__ uint64_t* nv_flag(const NvlsArgs& a, int owner, int ch, int ctr, int sender) {
  return a.fl[owner] + ((size_t)ch * kNvCounters + ctr) * kMaxRanks + sender;
}
__device__ __forceinline__ uint64_t* nv_base(const NvlsArgs& a, int ch) {
  return a.fl[a.me] + (size_t)a.nch * kNvCounters * kMaxRanks + ch;  // a.nch is the comm's fixed channel count
}

// warp 0: wait until my (ch, ctr) word of every sender in `who` (lane-indexed list of n ranks) reaches tg
__device__ bool nv_wait(const NvlsArgs& a, int ch, int ctr, const int* who, int n, int skip, uint64_t tg) {
  const int lane = threadIdx.x & 31;
  bool ok = true;
  if (lane < n && lane != skip) {
    const uint64_t* w = nv_flag(a, a.me, ch, ctr, who[lane]);
    const uint64_t t0 = [] { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }();
    uint32_t spins = 0;
    while (nv_ld_acquire(w) < tg) {
      if ((++spins & 1023u) == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if ((long long)(t - t0) > a.timeout_ns) {
          atomicOr(a.err, 1ull + ((unsigned long long)(16 + ctr) << 8) + ((unsigned long long)who[lane] << 16));
          ok = false;
          break;
        }
      }
    }
  }
  return __all_sync(0xffffffffu, ok);
}
// warp 0 (after the CTA's stores and a __syncthreads): release, then +1 on (owner, ch, ctr, me)
__device__ void nv_signal(const NvlsArgs& a, int ch, int ctr, const int* who, int n, int skip) {
  const int lane = threadIdx.x & 31;
  nv_fence();
  if (lane < n && lane != skip) nv_red(nv_flag(a, who[lane], ch, ctr, a.me));
}

// W: 16-bit dtype staged through an fp32 uc (a group of V elements = 16 bytes of x = UB = 32 bytes of uc)
//
// Software pipeline over the op's chunks (kNvSlots chunk slots in uc and in the cross slots): iteration it runs
//   P0 copy-in of chunk it            -> signal N_IN  (domain members)
//   P1 of chunk it-1: wait N_IN (all members) and, for slot reuse, N_XACK of chunk it-1-kNvSlots (cross
//      receivers); multimem.ld_reduce of my segment = the domain partial -> member i of every domain's cross
//      slot -> signal N_X
//   P2 of chunk it-2: wait N_X, and N_DONE of chunk it-2-kNvSlots (every member copied that slot out before my
//      multicast store overwrites it); fold the D partials, multimem.st -> signal N_XACK, N_OUT
//   P3 of chunk it-3: wait N_OUT; copy-out -> signal N_DONE
// Every wait is on signals peers send at an earlier iteration, so with all CTAs co-resident no cycle exists; a
// chunk's uc slot is refilled (P0, iteration g) only after this rank's P3 of the slot's previous chunk
// (iteration g-kNvSlots+3), which waited for every member's multicast store of it. Zero copy (send == recv == uc):
// chunk g lives at its own place in uc, no slot is reused.
template <int DT, bool W>
__global__ void __launch_bounds__(kNvThreads) k_nvls_allreduce(NvlsArgs a) {
  using VV = NvVec<DT>;
  constexpr int V = VV::V;
  constexpr int ES = 16 / V;
  constexpr size_t UB = W ? 32 : 16;  // uc / mc bytes per group
  static_assert(!W || DT != DT_F32, "fp32 staging is for 16-bit dtypes");
  using F32 = NvVec<DT_F32>;
  auto widen_st = [&](char* dst, const uint4& w, bool multi) {  // W: one 16-bit group -> two fp32 vectors
    uint4 lo, hi;
#pragma unroll
    for (int e = 0; e < 4; e++) {
      F32::set(lo, e, VV::get(w, e));
      F32::set(hi, e, VV::get(w, e + 4));
    }
    if (multi) {
      mc_st(dst, lo);
      mc_st(dst + 16, hi);
    } else {
      nv_st(dst, lo);
      nv_st(dst + 16, hi);
    }
  };
  auto narrow2 = [&](const uint4& lo, const uint4& hi) {  // two fp32 vectors -> one 16-bit group (RNE)
    uint4 w;
#pragma unroll
    for (int e = 0; e < 4; e++) {
      VV::set(w, e, F32::get(lo, e));
      VV::set(w, e + 4, F32::get(hi, e));
    }
    return w;
  };
  const int ch = blockIdx.x;
  const int tid = threadIdx.x, nth = blockDim.x;
  __shared__ int s_abort;
  __shared__ uint64_t s_base;
  if (tid == 0) {
    s_abort = 0;
    s_base = *nv_base(a, ch);
  }
  __syncthreads();
  const uint64_t base = s_base;
  const size_t nchunks = (a.count + a.ce - 1) / a.ce;
  // every chunk of an op uses the partition of its first chunk (a short last chunk only clips it), so a uc
  // vector always belongs to the same channel (q30)
  const size_t seg = ((min(a.ce, a.count) + V - 1) / V + a.d - 1) / a.d;  // vectors per segment
  const size_t sub = (seg + a.nch - 1) / a.nch;                         // vectors per channel per segment
  const size_t slot_b = (size_t)a.ce / V * UB;                           // uc bytes per chunk slot
  auto chunk_len = [&](size_t g) { return min(a.ce, a.count - g * a.ce); };
  auto range = [&](size_t nvec, int s, size_t& lo, size_t& hi) {
    const size_t s0 = (size_t)s * seg;
    lo = min(nvec, s0 + min(seg, (size_t)ch * sub));
    hi = min(nvec, s0 + min(seg, (size_t)(ch + 1) * sub));
  };
  auto ucp = [&](size_t g) { return (a.zero_copy ? g : g % kNvSlots) * slot_b; };  // chunk g's offset in uc / mc
  auto warp0_wait = [&](int ctr, const int* who, int n, int skip, uint64_t tg) {
    if (tid < 32 && !nv_wait(a, ch, ctr, who, n, skip, tg)) s_abort = 1;
  };
  const long long nit = nchunks ? (long long)nchunks + 3 : 0;
  for (long long it = 0; it < nit; ++it) {
    // ---- P0: x -> uc (every segment's channel range), zero padding past len ----
    if (it < (long long)nchunks) {
      const size_t g = (size_t)it, c0 = g * a.ce, len = chunk_len(g), nvec = (len + V - 1) / V;
      char* uc = a.uc + ucp(g);
      if (!a.zero_copy) {
        for (int sg = 0; sg < a.d; sg++) {
          size_t lo, hi;
          range(nvec, sg, lo, hi);
          for (size_t v = lo + tid; v < hi; v += nth) {
            uint4 w;
            if ((v + 1) * V <= len) {
              w = nv_ld(a.send + (c0 + v * V) * ES);
            } else {
              w = make_uint4(0, 0, 0, 0);
              for (int e = 0; e < V && v * V + e < len; e++) {
                if (ES == 4) (&w.x)[e] = *(const uint32_t*)(a.send + (c0 + v * V + e) * 4);
                else reinterpret_cast<uint16_t*>(&w)[e] = *(const uint16_t*)(a.send + (c0 + v * V + e) * 2);
              }
            }
            if (W) widen_st(uc + v * UB, w, false);
            else nv_st(uc + v * UB, w);
          }
        }
        // every storing thread orders its unicast stores before the peers' reads through the multicast alias (q31)
        nv_fence();
      }
      __syncthreads();
      if (tid < 32) nv_signal(a, ch, N_IN, a.dmem, a.d, a.i);
    }
    // ---- P1: domain partial through the switch -> member i of every domain's cross slot ----
    if (it >= 1 && it - 1 < (long long)nchunks) {
      const size_t g = (size_t)(it - 1), nvec = (chunk_len(g) + V - 1) / V;
      const uint64_t G = base + g;
      warp0_wait(N_IN, a.dmem, a.d, a.i, G + 1);
      if (a.D > 1 && g >= (size_t)kNvSlots) warp0_wait(N_XACK, a.xrank, a.D, a.k, G + 1 - kNvSlots);
      __syncthreads();
      if (s_abort) break;
      asm volatile("fence.proxy.alias;" ::: "memory");
      const char* mc = a.mc + ucp(g);
      const size_t so = (g % kNvSlots) * a.D;  // cross-slot base (units of xs_slot) of this chunk
      size_t lo, hi;
      range(nvec, a.i, lo, hi);
      // kNvUnroll switch reductions in flight per thread (each is a round trip through the NVSwitch)
      for (size_t v0 = lo + tid; v0 < hi; v0 += (size_t)kNvUnroll * nth) {
        uint4 p[kNvUnroll], p2[kNvUnroll];
#pragma unroll
        for (int u = 0; u < kNvUnroll; u++) {
          const size_t v = v0 + (size_t)u * nth;
          if (v >= hi) continue;
          if (W) {
            p[u] = mc_ld_reduce<DT_F32>(mc + v * UB);
            p2[u] = mc_ld_reduce<DT_F32>(mc + v * UB + 16);
          } else {
            p[u] = mc_ld_reduce<DT>(mc + v * UB);
          }
        }
#pragma unroll
        for (int u = 0; u < kNvUnroll; u++) {
          const size_t v = v0 + (size_t)u * nth;
          if (v >= hi) continue;
          const uint4 w = W ? narrow2(p[u], p2[u]) : p[u];
          const size_t off = (v - (size_t)a.i * seg) * 16;
          for (int q = 0; q < a.D; q++) nv_st(a.xs[q] + (so + a.k) * a.xs_slot + off, w);
        }
      }
      __syncthreads();
      if (tid < 32 && a.D > 1) nv_signal(a, ch, N_X, a.xrank, a.D, a.k);
    }
    // ---- P2: fold the D partials in ascending domain id, narrow once, multicast store ----
    if (it >= 2 && it - 2 < (long long)nchunks) {
      const size_t g = (size_t)(it - 2), nvec = (chunk_len(g) + V - 1) / V;
      const uint64_t G = base + g;
      if (a.D > 1) warp0_wait(N_X, a.xrank, a.D, a.k, G + 1);
      if (!a.zero_copy && g >= (size_t)kNvSlots) warp0_wait(N_DONE, a.dmem, a.d, -1, G + 1 - kNvSlots);
      __syncthreads();
      if (s_abort) break;
      char* mc = a.mc + ucp(g);
      const char* mine = a.xs[a.k] + (g % kNvSlots) * a.D * a.xs_slot;
      size_t lo, hi;
      range(nvec, a.i, lo, hi);
      for (size_t v = lo + tid; v < hi; v += nth) {
        const size_t off = (v - (size_t)a.i * seg) * 16;
        uint4 w = nv_ld(mine + off);
        if (a.D > 1) {
          float acc[V];
#pragma unroll
          for (int e = 0; e < V; e++) acc[e] = VV::get(w, e);
          for (int q = 1; q < a.D; q++) {
            const uint4 u = nv_ld(mine + (size_t)q * a.xs_slot + off);
#pragma unroll
            for (int e = 0; e < V; e++) acc[e] = __fadd_rn(acc[e], VV::get(u, e));
          }
#pragma unroll
          for (int e = 0; e < V; e++) VV::set(w, e, acc[e]);
        }
        if (W) widen_st(mc + v * UB, w, true);
        else mc_st(mc + v * UB, w);
      }
      __syncthreads();
      if (tid < 32) {
        if (a.D > 1) nv_signal(a, ch, N_XACK, a.xrank, a.D, a.k);
        nv_signal(a, ch, N_OUT, a.dmem, a.d, a.i);
      }
    }
    // ---- P3: uc -> y ----
    if (it >= 3) {
      const size_t g = (size_t)(it - 3), c0 = g * a.ce, len = chunk_len(g), nvec = (len + V - 1) / V;
      const uint64_t G = base + g;
      warp0_wait(N_OUT, a.dmem, a.d, a.i, G + 1);
      __syncthreads();
      if (s_abort) break;
      asm volatile("fence.proxy.alias;" ::: "memory");
      if (!a.zero_copy) {
        const char* uc = a.uc + ucp(g);
        for (int sg = 0; sg < a.d; sg++) {
          size_t l2, h2;
          range(nvec, sg, l2, h2);
          for (size_t v = l2 + tid; v < h2; v += nth) {
            const uint4 w = W ? narrow2(nv_ld(uc + v * UB), nv_ld(uc + v * UB + 16)) : nv_ld(uc + v * UB);
            if ((v + 1) * V <= len) {
              nv_st(a.recv + (c0 + v * V) * ES, w);
            } else {
              for (int e = 0; e < V && v * V + e < len; e++) {
                if (ES == 4) *(uint32_t*)(a.recv + (c0 + v * V + e) * 4) = (&w.x)[e];
                else *(uint16_t*)(a.recv + (c0 + v * V + e) * 2) = reinterpret_cast<const uint16_t*>(&w)[e];
              }
            }
          }
        }
      }
      __syncthreads();  // this slot's copy-out is done: members may multicast-store the slot's next chunk
      if (tid < 32) nv_signal(a, ch, N_DONE, a.dmem, a.d, -1);
    }
  }
  __syncthreads();
  if (tid == 0 && !s_abort) *nv_base(a, ch) = base + nchunks;
}

// ---------------------------------------------------------------- host: driver entry points -------
#define NV_FN(name) decltype(&::name) p_##name = nullptr
struct Drv {
  NV_FN(cuDeviceGet);
  NV_FN(cuDeviceGetAttribute);
  NV_FN(cuMulticastCreate);
  NV_FN(cuMulticastAddDevice);
  NV_FN(cuMulticastBindMem);
  NV_FN(cuMulticastUnbind);
  NV_FN(cuMulticastGetGranularity);
  NV_FN(cuMemCreate);
  NV_FN(cuMemRelease);
  NV_FN(cuMemAddressReserve);
  NV_FN(cuMemAddressFree);
  NV_FN(cuMemMap);
  NV_FN(cuMemUnmap);
  NV_FN(cuMemSetAccess);
  NV_FN(cuMemGetAllocationGranularity);
  NV_FN(cuMemExportToShareableHandle);
  NV_FN(cuMemImportFromShareableHandle);
  bool ok = false;
};
#undef NV_FN

Drv& drv() {
  static Drv d;
  static bool tried = false;
  if (tried) return d;
  tried = true;
  bool ok = true;
  auto get = [&](const char* sym, void** fn) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(sym, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !*fn)
      ok = false;
  };
#define NV_GET(name) get(#name, (void**)&d.p_##name)
  NV_GET(cuDeviceGet);
  NV_GET(cuDeviceGetAttribute);
  NV_GET(cuMulticastCreate);
  NV_GET(cuMulticastAddDevice);
  NV_GET(cuMulticastBindMem);
  NV_GET(cuMulticastUnbind);
  NV_GET(cuMulticastGetGranularity);
  NV_GET(cuMemCreate);
  NV_GET(cuMemRelease);
  NV_GET(cuMemAddressReserve);
  NV_GET(cuMemAddressFree);
  NV_GET(cuMemMap);
  NV_GET(cuMemUnmap);
  NV_GET(cuMemSetAccess);
  NV_GET(cuMemGetAllocationGranularity);
  NV_GET(cuMemExportToShareableHandle);
  NV_GET(cuMemImportFromShareableHandle);
#undef NV_GET
  d.ok = ok;
  return d;
}

struct McShared {  // one multicast object per domain, released with its last member
  CUmemGenericAllocationHandle h = 0;
  size_t bytes = 0;
  int refs = 0;
};

}  // namespace

struct NvlsState {
  int dev = 0, rank = 0, nch = 0;
  int wide = 1;              // HETCCL_NVLS_WIDE: 16-bit dtypes staged in fp32 (R7-gate accuracy)
  size_t bytes = 0;          // uc / mc bytes
  size_t ce_bytes = 0;       // chunk bytes per rank (multiple of 16 * d)
  CUmemGenericAllocationHandle uc_h = 0;
  CUdeviceptr uc = 0, mc = 0;
  McShared* mcs = nullptr;
  char* xs = nullptr;        // cross slots [2][D][ce/d] (cudaMalloc)
  uint64_t* fl = nullptr;    // flags [nch][4][kMaxRanks] + base[nch] (cudaMalloc, zeroed)
  // one rank per process (nvls_proc_*): the domain leader's listening socket and exported multicast handle,
  // and the peers' xs / fl as opened through CUDA IPC
  int listen_fd = -1, mc_fd = -1;
  bool mc_imported = false;
  char* peer_xs[kMaxRanks] = {nullptr};
  uint64_t* peer_fl[kMaxRanks] = {nullptr};
  bool peer_ipc[kMaxRanks] = {false};
  bool joint = false;        // xs and fl are one allocation (one-rank-per-process set-up)
  size_t gran = 0;
  NvlsArgs tmpl{};           // peers, topology (pointers filled at create)
};

static void nv_err(char* err, size_t len, const char* what, int r) {
  if (err && len) snprintf(err, len, "NVLS: %s failed (%d)", what, r);
}

int nvls_eligible_topo(const Topo& t) {
  if (t.n < 2) return 0;
  const int d = t.dom_size[0];
  if (d < 2) return 0;
  for (int k = 1; k < t.D; k++)
    if (t.dom_size[k] != d) return 0;
  return 1;
}

void nvls_destroy(NvlsState* s) {
  if (!s) return;
  Drv& D = drv();
  int prev;
  cudaGetDevice(&prev);
  cudaSetDevice(s->dev);
  cudaDeviceSynchronize();
  if (s->mc) {
    D.p_cuMemUnmap(s->mc, s->bytes);
    D.p_cuMemAddressFree(s->mc, s->bytes);
  }
  if (s->uc) {
    D.p_cuMemUnmap(s->uc, s->bytes);
    D.p_cuMemAddressFree(s->uc, s->bytes);
  }
  if (s->mcs && s->mcs->h) {
    CUdevice cd;
    if (D.p_cuDeviceGet(&cd, s->dev) == CUDA_SUCCESS) D.p_cuMulticastUnbind(s->mcs->h, cd, 0, s->bytes);
  }
  if (s->uc_h) D.p_cuMemRelease(s->uc_h);
  if (s->mcs && --s->mcs->refs == 0) {
    if (s->mcs->h) D.p_cuMemRelease(s->mcs->h);
    delete s->mcs;
  }
  for (int r = 0; r < kMaxRanks; r++) {
    if (!s->peer_ipc[r]) continue;
    if (s->peer_xs[r]) cudaIpcCloseMemHandle(s->peer_xs[r]);
  }
  if (s->xs) cudaFree(s->xs);
  if (s->fl && !s->joint) cudaFree(s->fl);
  if (s->listen_fd >= 0) close(s->listen_fd);
  if (s->mc_fd >= 0) close(s->mc_fd);
  cudaSetDevice(prev);
  delete s;
}

// every rank of a single-process communicator (devs[r] = device of rank r); out[r] = its state
int nvls_create(int n, const int* devs, const Topo& t, size_t bytes_per_rank, int nch, NvlsState** out, char* err,
                size_t errlen) {
  for (int r = 0; r < n; r++) out[r] = nullptr;
  if (!nvls_eligible_topo(t)) {
    nv_err(err, errlen, "domain sizes must be equal and >= 2", 0);
    return 1;
  }
  Drv& D = drv();
  if (!D.ok) {
    nv_err(err, errlen, "driver entry points", 0);
    return 1;
  }
  int prev;
  cudaGetDevice(&prev);
  const int d = t.dom_size[0];
  int rc = 0;
  for (int r = 0; r < n && !rc; r++) {
    CUdevice cd;
    int sup = 0;
    if (D.p_cuDeviceGet(&cd, devs[r]) != CUDA_SUCCESS ||
        D.p_cuDeviceGetAttribute(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd) != CUDA_SUCCESS || !sup) {
      nv_err(err, errlen, "multicast not supported on this device", devs[r]);
      rc = 1;
    }
  }
  if (rc) return rc;
  // sizes: a multiple of the multicast and allocation granularities; chunk = bytes (16 * d aligned)
  CUmulticastObjectProp mp{};
  mp.numDevices = (unsigned)d;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes_per_rank;
  size_t mg = 0, ag = 0;
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = devs[0];
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  if ((rc = D.p_cuMulticastGetGranularity(&mg, &mp, CU_MULTICAST_GRANULARITY_MINIMUM)) ||
      (rc = D.p_cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM))) {
    nv_err(err, errlen, "granularity", rc);
    return 1;
  }
  const size_t gran = std::max(mg, ag);
  const size_t bytes = (std::max(bytes_per_rank, (size_t)1) + gran - 1) / gran * gran;
  const size_t unit = (size_t)16 * d;
  const size_t ce_bytes = bytes / unit * unit;
  const size_t xs_slot = ce_bytes / d;
  for (int r = 0; r < n; r++) {
    out[r] = new NvlsState();
    out[r]->dev = devs[r];
    out[r]->rank = r;
    out[r]->nch = nch;
    out[r]->bytes = bytes;
    out[r]->ce_bytes = ce_bytes;
    const char* w = getenv("HETCCL_NVLS_WIDE");
    out[r]->wide = !(w && *w == '0');
  }
  auto fail = [&](const char* what, int code) {
    nv_err(err, errlen, what, code);
    for (int r = 0; r < n; r++) {
      nvls_destroy(out[r]);
      out[r] = nullptr;
    }
    cudaSetDevice(prev);
    return 1;
  };
  // one multicast object per domain; add every member's device before binding memory
  for (int k = 0; k < t.D; k++) {
    McShared* m = new McShared();
    m->bytes = bytes;
    mp.size = bytes;
    if ((rc = D.p_cuMulticastCreate(&m->h, &mp))) {
      delete m;
      return fail("cuMulticastCreate", rc);
    }
    for (int j = 0; j < d; j++) {
      const int r = t.members[t.dom_first[k] + j];
      out[r]->mcs = m;
      m->refs++;
      CUdevice cd;
      D.p_cuDeviceGet(&cd, devs[r]);
      if ((rc = D.p_cuMulticastAddDevice(m->h, cd))) return fail("cuMulticastAddDevice", rc);
    }
  }
  for (int r = 0; r < n; r++) {
    NvlsState* s = out[r];
    cudaSetDevice(s->dev);
    cudaFree(0);
    CUmemAllocationProp p = ap;
    p.location.id = s->dev;
    if ((rc = D.p_cuMemCreate(&s->uc_h, bytes, &p, 0))) return fail("cuMemCreate", rc);
    if ((rc = D.p_cuMulticastBindMem(s->mcs->h, 0, s->uc_h, 0, bytes, 0))) return fail("cuMulticastBindMem", rc);
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = s->dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if ((rc = D.p_cuMemAddressReserve(&s->uc, bytes, gran, 0, 0))) return fail("cuMemAddressReserve(uc)", rc);
    if ((rc = D.p_cuMemMap(s->uc, bytes, 0, s->uc_h, 0))) return fail("cuMemMap(uc)", rc);
    if ((rc = D.p_cuMemSetAccess(s->uc, bytes, &acc, 1))) return fail("cuMemSetAccess(uc)", rc);
    if ((rc = D.p_cuMemAddressReserve(&s->mc, bytes, gran, 0, 0))) return fail("cuMemAddressReserve(mc)", rc);
    if ((rc = D.p_cuMemMap(s->mc, bytes, 0, s->mcs->h, 0))) return fail("cuMemMap(mc)", rc);
    if ((rc = D.p_cuMemSetAccess(s->mc, bytes, &acc, 1))) return fail("cuMemSetAccess(mc)", rc);
    if (cudaMalloc((void**)&s->xs, 2 * (size_t)t.D * xs_slot) != cudaSuccess) return fail("cudaMalloc(xs)", 0);
    const size_t flb = ((size_t)nch * kNvCounters * kMaxRanks + nch) * sizeof(uint64_t);
    if (cudaMalloc((void**)&s->fl, flb) != cudaSuccess || cudaMemset(s->fl, 0, flb) != cudaSuccess)
      return fail("cudaMalloc(flags)", 0);
    if (cudaMemset((void*)s->uc, 0, bytes) != cudaSuccess) return fail("cudaMemset(uc)", 0);
    if (cudaDeviceSynchronize() != cudaSuccess) return fail("cudaDeviceSynchronize", 0);
  }
  for (int r = 0; r < n; r++) {
    NvlsState* s = out[r];
    NvlsArgs& a = s->tmpl;
    memset(&a, 0, sizeof(a));
    a.me = r;
    a.d = d;
    a.D = t.D;
    a.i = t.rank_idx[r];
    a.k = t.rank_dom[r];
    a.nch = nch;
    a.ce = 0;  // per dtype at launch
    a.xs_slot = xs_slot;
    a.uc = (char*)s->uc;
    a.mc = (char*)s->mc;
    for (int j = 0; j < d; j++) a.dmem[j] = t.members[t.dom_first[a.k] + j];
    for (int q = 0; q < t.D; q++) {
      const int x = t.members[t.dom_first[q] + a.i];
      a.xrank[q] = x;
      a.xs[q] = out[x]->xs;
    }
    for (int p = 0; p < n; p++) a.fl[p] = out[p]->fl;
  }
  cudaSetDevice(prev);
  return 0;
}

// 1 if [p, p+bytes) overlaps the uc buffer while 16-bit data would be staged wide through it (the copy-in
// would overwrite its own input): the caller rejects that (hetcclInvalidArgument)
int nvls_aliases_staging(const NvlsState* s, int dt, const void* p, size_t bytes) {
  if (!s || !s->wide || dtype_size(dt) != 2 || !p) return 0;
  const uintptr_t a0 = (uintptr_t)p, u0 = (uintptr_t)s->uc;
  return a0 < u0 + s->bytes && u0 < a0 + bytes;
}

// ---------------------------------------------------------------- one rank per process ----------
namespace {
long long now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (long long)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}
// wait until fd is readable (or writable), at most until the deadline
bool wait_fd(int fd, short ev, long long deadline) {
  for (;;) {
    const long long left = deadline - now_ns();
    if (left <= 0) return false;
    pollfd p{fd, ev, 0};
    const int r = poll(&p, 1, (int)std::min<long long>(left / 1000000 + 1, 1000));
    if (r > 0) return true;
    if (r < 0) return false;
  }
}
bool send_byte(int fd, char c, int pass_fd = -1) {
  iovec io{&c, 1};
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  char ctl[CMSG_SPACE(sizeof(int))];
  if (pass_fd >= 0) {
    memset(ctl, 0, sizeof(ctl));
    m.msg_control = ctl;
    m.msg_controllen = sizeof(ctl);
    cmsghdr* cm = CMSG_FIRSTHDR(&m);
    cm->cmsg_level = SOL_SOCKET;
    cm->cmsg_type = SCM_RIGHTS;
    cm->cmsg_len = CMSG_LEN(sizeof(int));
    memcpy(CMSG_DATA(cm), &pass_fd, sizeof(int));
  }
  return sendmsg(fd, &m, 0) == 1;
}
// receive one byte (and a passed file descriptor, if any) before the deadline
bool recv_byte(int fd, char want, long long deadline, int* got_fd = nullptr) {
  if (!wait_fd(fd, POLLIN, deadline)) return false;
  char c = 0;
  iovec io{&c, 1};
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  char ctl[CMSG_SPACE(sizeof(int))];
  memset(ctl, 0, sizeof(ctl));
  m.msg_control = ctl;
  m.msg_controllen = sizeof(ctl);
  if (recvmsg(fd, &m, 0) != 1 || c != want) return false;
  if (got_fd) {
    cmsghdr* cm = CMSG_FIRSTHDR(&m);
    if (!cm || cm->cmsg_type != SCM_RIGHTS) return false;
    memcpy(got_fd, CMSG_DATA(cm), sizeof(int));
  }
  return true;
}
sockaddr_un abstract_addr(const char* name, socklen_t* len) {
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  a.sun_path[0] = 0;  // abstract namespace: no file, gone with the socket
  strncpy(a.sun_path + 1, name, sizeof(a.sun_path) - 2);
  *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + strlen(name));
  return a;
}
// uc: this device's memory bound to the multicast object, mapped at uc; mc: the multicast address
int bind_and_map(NvlsState* s, char* err, size_t errlen) {
  Drv& D = drv();
  CUmemAllocationProp p{};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = s->dev;
  p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  int rc;
  if ((rc = D.p_cuMemCreate(&s->uc_h, s->bytes, &p, 0))) return nv_err(err, errlen, "cuMemCreate", rc), 1;
  if ((rc = D.p_cuMulticastBindMem(s->mcs->h, 0, s->uc_h, 0, s->bytes, 0)))
    return nv_err(err, errlen, "cuMulticastBindMem", rc), 1;
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = s->dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if ((rc = D.p_cuMemAddressReserve(&s->uc, s->bytes, s->gran, 0, 0))) return nv_err(err, errlen, "reserve(uc)", rc), 1;
  if ((rc = D.p_cuMemMap(s->uc, s->bytes, 0, s->uc_h, 0))) return nv_err(err, errlen, "cuMemMap(uc)", rc), 1;
  if ((rc = D.p_cuMemSetAccess(s->uc, s->bytes, &acc, 1))) return nv_err(err, errlen, "cuMemSetAccess(uc)", rc), 1;
  if ((rc = D.p_cuMemAddressReserve(&s->mc, s->bytes, s->gran, 0, 0))) return nv_err(err, errlen, "reserve(mc)", rc), 1;
  if ((rc = D.p_cuMemMap(s->mc, s->bytes, 0, s->mcs->h, 0))) return nv_err(err, errlen, "cuMemMap(mc)", rc), 1;
  if ((rc = D.p_cuMemSetAccess(s->mc, s->bytes, &acc, 1))) return nv_err(err, errlen, "cuMemSetAccess(mc)", rc), 1;
  if (cudaMemset((void*)s->uc, 0, s->bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    return nv_err(err, errlen, "cudaMemset(uc)", 0), 1;
  return 0;
}
}  // namespace

int nvls_proc_begin(const Topo& t, int rank, int dev, size_t bytes_per_rank, int nch, NvlsState** out, NvlsBlob* blob,
                    char* err, size_t errlen) {
  *out = nullptr;
  memset(blob, 0, sizeof(*blob));
  if (!nvls_eligible_topo(t)) return nv_err(err, errlen, "domain sizes must be equal and >= 2", 0), 1;
  Drv& D = drv();
  if (!D.ok) return nv_err(err, errlen, "driver entry points", 0), 1;
  const int d = t.dom_size[0];
  CUdevice cd;
  int sup = 0;
  if (D.p_cuDeviceGet(&cd, dev) != CUDA_SUCCESS ||
      D.p_cuDeviceGetAttribute(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd) != CUDA_SUCCESS || !sup)
    return nv_err(err, errlen, "multicast not supported on this device", dev), 1;
  CUmulticastObjectProp mp{};
  mp.numDevices = (unsigned)d;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes_per_rank;
  size_t mg = 0, ag = 0;
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  int rc;
  if ((rc = D.p_cuMulticastGetGranularity(&mg, &mp, CU_MULTICAST_GRANULARITY_MINIMUM)) ||
      (rc = D.p_cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM)))
    return nv_err(err, errlen, "granularity", rc), 1;
  NvlsState* s = new NvlsState();
  s->dev = dev;
  s->rank = rank;
  s->nch = nch;
  s->gran = std::max(mg, ag);
  s->bytes = (std::max(bytes_per_rank, (size_t)1) + s->gran - 1) / s->gran * s->gran;
  s->ce_bytes = s->bytes / ((size_t)16 * d) * ((size_t)16 * d);
  const char* w = getenv("HETCCL_NVLS_WIDE");
  s->wide = !(w && *w == '0');
  s->joint = true;
  const size_t xs_bytes = (2 * (size_t)t.D * (s->ce_bytes / d) + 255) / 256 * 256;
  const size_t flb = ((size_t)nch * kNvCounters * kMaxRanks + nch) * sizeof(uint64_t);
  auto fail = [&](const char* what, int code) {
    nv_err(err, errlen, what, code);
    nvls_destroy(s);
    return 1;
  };
  if (cudaMalloc((void**)&s->xs, xs_bytes + flb) != cudaSuccess) return fail("cudaMalloc(xs, flags)", 0);
  s->fl = (uint64_t*)(s->xs + xs_bytes);
  if (cudaMemset(s->fl, 0, flb) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return fail("cudaMemset", 0);
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, s->xs) != cudaSuccess) return fail("cudaIpcGetMemHandle(xs)", 0);
  memcpy(blob->ipc, &h, sizeof(h));
  s->tmpl.xs_slot = s->ce_bytes / d;
  if (t.rank_idx[rank] == 0) {  // domain leader: the multicast object and the socket that hands it out
    s->mcs = new McShared();
    s->mcs->refs = 1;
    mp.size = s->bytes;
    if ((rc = D.p_cuMulticastCreate(&s->mcs->h, &mp))) return fail("cuMulticastCreate", rc);
    if ((rc = D.p_cuMulticastAddDevice(s->mcs->h, cd))) return fail("cuMulticastAddDevice", rc);
    if ((rc = D.p_cuMemExportToShareableHandle(&s->mc_fd, s->mcs->h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0)))
      return fail("cuMemExportToShareableHandle", rc);
    snprintf(blob->sock, sizeof(blob->sock), "hetccl-nvls-%d-%d-%llx", (int)getpid(), rank,
             (unsigned long long)now_ns());
    s->listen_fd = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    socklen_t len;
    sockaddr_un a = abstract_addr(blob->sock, &len);
    if (s->listen_fd < 0 || bind(s->listen_fd, (sockaddr*)&a, len) != 0 || listen(s->listen_fd, kMaxRanks) != 0)
      return fail("leader socket", errno);
  }
  blob->enabled = 1;
  *out = s;
  return 0;
}

int nvls_proc_connect(NvlsState* s, const Topo& t, int rank, const NvlsBlob* const* blobs, long long timeout_ns,
                      char* err, size_t errlen) {
  Drv& D = drv();
  const long long deadline = now_ns() + timeout_ns;
  const int k = t.rank_dom[rank], d = t.dom_size[k];
  const int leader = t.members[t.dom_first[k]];
  CUdevice cd;
  D.p_cuDeviceGet(&cd, s->dev);
  // every peer's cross slots + flags
  const size_t xs_bytes = (size_t)((char*)s->fl - s->xs);
  for (int r = 0; r < t.n; r++) {
    if (r == rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, blobs[r]->ipc, sizeof(h));
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
      return nv_err(err, errlen, "cudaIpcOpenMemHandle(nvls)", r), 1;
    s->peer_xs[r] = (char*)p;
    s->peer_fl[r] = (uint64_t*)((char*)p + xs_bytes);
    s->peer_ipc[r] = true;
  }
  if (rank == leader) {
    // hand the multicast handle to every member, wait until each added its device, then everyone binds
    int conns[kMaxRanks];
    int nc = 0;
    bool ok = true;
    for (; nc < d - 1 && ok; nc++) {
      ok = wait_fd(s->listen_fd, POLLIN, deadline);
      conns[nc] = ok ? accept4(s->listen_fd, nullptr, nullptr, SOCK_CLOEXEC) : -1;
      ok = ok && conns[nc] >= 0 && send_byte(conns[nc], 'F', s->mc_fd);
    }
    for (int i = 0; i < nc && ok; i++) ok = recv_byte(conns[i], 'A', deadline);
    for (int i = 0; i < nc && ok; i++) ok = send_byte(conns[i], 'B');
    ok = ok && bind_and_map(s, err, errlen) == 0;
    for (int i = 0; i < nc && ok; i++) ok = recv_byte(conns[i], 'C', deadline);
    for (int i = 0; i < nc && ok; i++) ok = send_byte(conns[i], 'D');
    for (int i = 0; i < nc; i++)
      if (conns[i] >= 0) close(conns[i]);
    if (!ok) return (err && !*err ? nv_err(err, errlen, "leader hand-off", 0) : (void)0), 1;
  } else {
    if (!blobs[leader]->sock[0]) return nv_err(err, errlen, "leader published no socket", leader), 1;
    socklen_t len;
    sockaddr_un a = abstract_addr(blobs[leader]->sock, &len);
    int fd = -1;
    while (fd < 0) {
      fd = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
      if (fd >= 0 && connect(fd, (sockaddr*)&a, len) == 0) break;
      if (fd >= 0) close(fd);
      fd = -1;
      if (now_ns() > deadline) return nv_err(err, errlen, "connect to leader", errno), 1;
      usleep(1000);
    }
    int mfd = -1;
    bool ok = recv_byte(fd, 'F', deadline, &mfd);
    if (ok) {
      s->mcs = new McShared();
      s->mcs->refs = 1;
      int rc = D.p_cuMemImportFromShareableHandle(&s->mcs->h, (void*)(uintptr_t)mfd,
                                                  CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
      close(mfd);
      ok = rc == CUDA_SUCCESS && D.p_cuMulticastAddDevice(s->mcs->h, cd) == CUDA_SUCCESS;
      if (!ok) nv_err(err, errlen, "import / add device", rc);
    }
    ok = ok && send_byte(fd, 'A') && recv_byte(fd, 'B', deadline);
    ok = ok && bind_and_map(s, err, errlen) == 0;
    ok = ok && send_byte(fd, 'C') && recv_byte(fd, 'D', deadline);
    close(fd);
    if (!ok) return (err && !*err ? nv_err(err, errlen, "member hand-off", 0) : (void)0), 1;
  }
  if (s->listen_fd >= 0) {
    close(s->listen_fd);
    s->listen_fd = -1;
  }
  // kernel arguments (as nvls_create's, with the peers' buffers as opened here)
  NvlsArgs& a = s->tmpl;
  const size_t xs_slot = a.xs_slot;
  memset(&a, 0, sizeof(a));
  a.me = rank;
  a.d = d;
  a.D = t.D;
  a.i = t.rank_idx[rank];
  a.k = k;
  a.nch = s->nch;
  a.xs_slot = xs_slot;
  a.uc = (char*)s->uc;
  a.mc = (char*)s->mc;
  for (int j = 0; j < d; j++) a.dmem[j] = t.members[t.dom_first[k] + j];
  for (int q = 0; q < t.D; q++) {
    const int x = t.members[t.dom_first[q] + a.i];
    a.xrank[q] = x;
    a.xs[q] = x == rank ? s->xs : s->peer_xs[x];
  }
  for (int p = 0; p < t.n; p++) a.fl[p] = p == rank ? s->fl : s->peer_fl[p];
  return 0;
}

void nvls_buffer(const NvlsState* s, void** p, size_t* bytes) {
  if (p) *p = s ? (void*)s->uc : nullptr;
  if (bytes) *bytes = s ? s->ce_bytes : 0;
}

// The path choice depends only on values every rank shares (dtype, op), never on a rank's own pointers:
// ranks that chose differently would wait on different flag arrays. Alignment is checked by the caller
// (run_op), which rejects unaligned buffers in NVLS mode instead of switching path.
int nvls_supports(const NvlsState* s, int dt, int red, const void*, const void*) {
  return s && red == RED_SUM && (dt == DT_BF16 || dt == DT_F16 || dt == DT_F32);
}

cudaError_t nvls_allreduce(NvlsState* s, const void* send, void* recv, size_t count, int dt,
                           unsigned long long* err, long long timeout_ns, cudaStream_t st) {
  NvlsArgs a = s->tmpl;
  const int es = dtype_size(dt);
  const bool wide = s->wide && es == 2;
  a.send = (const char*)send;
  a.recv = (char*)recv;
  a.count = count;
  // kNvSlots chunk slots in uc (uc holds fp32 when staging wide); slot bytes a multiple of 16 * d so every
  // segment starts on a vector
  const size_t unit = (size_t)16 * a.d;
  const size_t chunk_b = std::max(unit, s->ce_bytes / kNvSlots / unit * unit);
  a.ce = chunk_b / (wide ? 4 : es);  // elements per chunk
  const size_t V = (dt == DT_F32) ? 4 : 8;
  a.xs_slot = ((a.ce / V + a.d - 1) / a.d) * 16;  // one domain partial of one member's segment of a chunk
  a.err = err;
  a.timeout_ns = timeout_ns;
  a.wide = wide;
  a.zero_copy = !wide && send == recv && (const char*)send == (const char*)s->uc && count * es <= s->ce_bytes &&
                (count * es) % 16 == 0;
  dim3 grid(s->nch), block(kNvThreads);
  switch (dt) {
    case DT_BF16:
      if (wide) k_nvls_allreduce<DT_BF16, true><<<grid, block, 0, st>>>(a);
      else k_nvls_allreduce<DT_BF16, false><<<grid, block, 0, st>>>(a);
      break;
    case DT_F16:
      if (wide) k_nvls_allreduce<DT_F16, true><<<grid, block, 0, st>>>(a);
      else k_nvls_allreduce<DT_F16, false><<<grid, block, 0, st>>>(a);
      break;
    default: k_nvls_allreduce<DT_F32, false><<<grid, block, 0, st>>>(a); break;
  }
  return cudaGetLastError();
}

}  // namespace hetccl
