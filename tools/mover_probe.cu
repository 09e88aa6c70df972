// Mover probe: how fast can one CTA design stream a K-source fold into M destinations on one B200?
// Emulates the pipeline kernels' data movers (kernels.cu cta_fold / tma_move) outside the protocol:
// K bf16 sources of N bytes each are folded (fp32 add, one narrowing) and the result is stored to M
// destinations; CTA b works blocks b, b+G, ... of BLK bytes per operand, one mover call per block
// (the real kernels call a mover once per piece, so per-call prologues count).
//   impl ldg   : 16-byte register loads, U vectors per source in flight per thread
//   impl lgsts : cp.async (LDGSTS) staging of all K sources x U vectors, then fold (round-1 default),
//                plus an optional L2 bulk prefetch PF batches ahead
//   impl tma   : ring of NST shared-memory stages filled by cp.async.bulk (one producer thread),
//                chunk = vpt*128*16 bytes per operand, optional L2 bulk prefetch PF chunks beyond the ring
// Reports HBM traffic (K+M)*N over the kernel time. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mover_probe tools/mover_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e = (x);                                                                \
    if (e != cudaSuccess) {                                                             \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

constexpr int kMax = 10;
struct Args {
  const char* src[kMax];
  char* dst[kMax];
  int K, M;
  size_t N, BLK;  // bytes per operand; block bytes per operand
  int U, PF, NST, SB, VPT;
};

__device__ __forceinline__ uint4 ldcg(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void acc_add(float* a, const uint4& w, bool first) {
  const uint32_t x[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; i++) {
    float lo = __uint_as_float(x[i] << 16), hi = __uint_as_float(x[i] & 0xffff0000u);
    a[2 * i] = first ? lo : __fadd_rn(a[2 * i], lo);
    a[2 * i + 1] = first ? hi : __fadd_rn(a[2 * i + 1], hi);
  }
}
__device__ __forceinline__ uint4 pack(const float* a) {
  uint32_t o[4];
#pragma unroll
  for (int i = 0; i < 4; i++)
    o[i] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a[2 * i])) |
           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a[2 * i + 1])) << 16);
  return make_uint4(o[0], o[1], o[2], o[3]);
}
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---------------------------------------------------------------- ldg
template <int U>
__device__ void mv_ldg(const Args& a, size_t off, size_t nv) {
  const int tid = threadIdx.x, nth = blockDim.x;
  for (size_t v0 = tid; v0 < nv; v0 += (size_t)U * nth) {
    float acc[U][8];
    for (int k = 0; k < a.K; k++) {
      uint4 w[U];
#pragma unroll
      for (int u = 0; u < U; u++)
        if (v0 + u * nth < nv) w[u] = ldcg(a.src[k] + off + (v0 + u * nth) * 16);
#pragma unroll
      for (int u = 0; u < U; u++) acc_add(acc[u], w[u], k == 0);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (v0 + u * nth >= nv) continue;
      const uint4 o = pack(acc[u]);
      for (int m = 0; m < a.M; m++) stg(a.dst[m] + off + (v0 + u * nth) * 16, o);
    }
  }
}

// ---------------------------------------------------------------- ldgsts (+ L2 prefetch)
template <int U>
__device__ void mv_lgsts(const Args& a, size_t off, size_t nv, uint4* stage) {
  const int tid = threadIdx.x, nth = blockDim.x;
  for (size_t v0 = tid; v0 < nv; v0 += (size_t)U * nth) {
    if (a.PF > 0 && tid == 0) {
      const size_t vs = v0 + (size_t)a.PF * U * nth;
      if (vs < nv)
        for (int k = 0; k < a.K; k++)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.src[k] + off + vs * 16),
                       "r"((uint32_t)(min((size_t)U * nth, nv - vs) * 16))
                       : "memory");
    }
    for (int k = 0; k < a.K; k++)
#pragma unroll
      for (int u = 0; u < U; u++)
        if (v0 + u * nth < nv)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(&stage[(k * U + u) * nth + tid])),
                       "l"(a.src[k] + off + (v0 + u * nth) * 16)
                       : "memory");
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    float acc[U][8];
    for (int k = 0; k < a.K; k++)
#pragma unroll
      for (int u = 0; u < U; u++) acc_add(acc[u], stage[(k * U + u) * nth + tid], k == 0);
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (v0 + u * nth >= nv) continue;
      const uint4 o = pack(acc[u]);
      for (int m = 0; m < a.M; m++) stg(a.dst[m] + off + (v0 + u * nth) * 16, o);
    }
  }
}

// ---------------------------------------------------------------- tma ring
__shared__ __align__(8) uint64_t s_full[16];
__shared__ unsigned s_seq;
__device__ void mv_tma(const Args& a, size_t off, size_t nv, unsigned char* ring) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int NST = a.NST;
  int vpt = a.SB / (a.K * 16 * nth);
  if (vpt > a.VPT) vpt = a.VPT;
  const size_t cv = (size_t)vpt * nth;
  const uint32_t chb = (uint32_t)cv * 16;
  const size_t nch = (nv + cv - 1) / cv;
  const unsigned seq0 = *(volatile unsigned*)&s_seq;
  auto issue = [&](size_t c) {
    const unsigned g = seq0 + (unsigned)c;
    const int s = g % NST;
    const size_t v0 = c * cv;
    const uint32_t bytes = (uint32_t)(min(cv, nv - v0) * 16);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&s_full[s])), "r"(bytes * a.K)
                 : "memory");
    for (int k = 0; k < a.K; k++)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(ring + (size_t)s * a.SB + (size_t)k * chb)),
                   "l"(a.src[k] + off + v0 * 16), "r"(bytes), "r"(sa(&s_full[s]))
                   : "memory");
    if (a.PF > 0) {
      const size_t vp = (c + a.PF) * cv;
      if (vp < nv)
        for (int k = 0; k < a.K; k++)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.src[k] + off + vp * 16),
                       "r"((uint32_t)(min(cv, nv - vp) * 16))
                       : "memory");
    }
  };
  if (tid == 0)
    for (size_t c = 0; c < nch && c < (size_t)NST - 1; c++) issue(c);
  for (size_t c = 0; c < nch; c++) {
    if (tid == 0 && c + NST - 1 < nch) issue(c + NST - 1);
    const unsigned g = seq0 + (unsigned)c;
    const int s = g % NST;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok)
                   : "r"(sa(&s_full[s])), "r"((g / NST) & 1u)
                   : "memory");
    const unsigned char* st = ring + (size_t)s * a.SB;
    for (int u = 0; u < vpt; u++) {
      const size_t idx = (size_t)u * nth + tid, v = c * cv + idx;
      if (v >= nv) break;
      float acc[8];
      for (int k = 0; k < a.K; k++) acc_add(acc, *(const uint4*)(st + (size_t)k * chb + idx * 16), k == 0);
      const uint4 o = pack(acc);
      for (int m = 0; m < a.M; m++) stg(a.dst[m] + off + v * 16, o);
    }
    __syncthreads();
  }
  *(volatile unsigned*)&s_seq = seq0 + (unsigned)nch;
}

// ---------------------------------------------------------------- tma2: the library's mover (full/empty
// mbarriers, no CTA barrier per chunk, evict_first hints); S2G=1 stores results with bulk copies from shared
__shared__ __align__(8) uint64_t s_empty[16];
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(sa(b)), "r"(par)
                 : "memory");
}
template <int S2G>
__device__ void mv_tma2(const Args& a, size_t off, size_t nv_, unsigned char* ring) {
  const int tid = threadIdx.x, nth = blockDim.x, NST = a.NST, lane = tid & 31;
  const uint32_t nv = (uint32_t)nv_;
  const uint32_t cv = min((uint32_t)(a.SB / (a.K * 16)) / 8 * 8, (uint32_t)(4 * nth));
  const uint32_t chb = cv * 16, nch = (nv + cv - 1) / cv;
  const unsigned seq0 = *(volatile unsigned*)&s_seq;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](uint32_t cn) {
    const unsigned g = seq0 + cn, st = g % NST, u = g / NST;
    if (u > 0) mwait(&s_empty[st], (u - 1) & 1u);
    if (S2G && u > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    const uint32_t bytes = min(cv, nv - cn * cv) * 16;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&s_full[st])), "r"(bytes * a.K) : "memory");
    for (int k = 0; k < a.K; k++)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
              sa(ring + (size_t)st * a.SB + (size_t)k * chb)),
          "l"(a.src[k] + off + (size_t)cn * chb), "r"(bytes), "r"(sa(&s_full[st])), "l"(pol)
          : "memory");
  };
  if (tid == 0)
    for (uint32_t c = 0; c < nch && c < (uint32_t)NST - 1; c++) issue(c);
  for (uint32_t c = 0; c < nch; c++) {
    if (tid == 0 && c + NST - 1 < nch) issue(c + NST - 1);
    const unsigned g = seq0 + c, st = g % NST;
    mwait(&s_full[st], (g / NST) & 1u);
    unsigned char* sb = ring + (size_t)st * a.SB;
    const uint32_t lim = min(cv, nv - c * cv);
    for (uint32_t idx = tid; idx < lim; idx += nth) {
      float acc[8];
      acc_add(acc, *(const uint4*)(sb + idx * 16), true);
#pragma unroll 1
      for (int k = 1; k < a.K; k++) acc_add(acc, *(const uint4*)(sb + k * chb + idx * 16), false);
      const uint4 o = a.K == 1 ? *(const uint4*)(sb + idx * 16) : pack(acc);
      if (S2G) *(uint4*)(sb + idx * 16) = o;
      else
        for (int m = 0; m < a.M; m++)
          asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a.dst[m] + off + ((size_t)c * cv + idx) * 16),
                       "r"(o.x), "r"(o.y), "r"(o.z), "r"(o.w), "l"(pol)
                       : "memory");
    }
    if (S2G) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();  // every result of the chunk is in shared memory
      if (tid == 0) {
        for (int m = 0; m < a.M; m++)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                           a.dst[m] + off + (size_t)c * chb),
                       "r"(sa(sb)), "r"(lim * 16), "l"(pol)
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&s_empty[st])) : "memory");
  }
  if (S2G && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  *(volatile unsigned*)&s_seq = seq0 + nch;
}

template <int IMPL, int U>
__global__ void __launch_bounds__(128) k_probe(const __grid_constant__ Args a) {
  extern __shared__ __align__(128) unsigned char dyn[];
  if (IMPL >= 2) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < a.NST; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&s_full[s])));
      for (int s = 0; s < a.NST; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(sa(&s_empty[s])));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      s_seq = 0;
    }
    __syncthreads();
  }
  const size_t nblk = a.N / a.BLK;
  for (size_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    const size_t off = b * a.BLK, nv = a.BLK / 16;
    if (IMPL == 0) mv_ldg<U>(a, off, nv);
    else if (IMPL == 1) mv_lgsts<U>(a, off, nv, (uint4*)dyn);
    else if (IMPL == 2) mv_tma(a, off, nv, dyn);
    else if (IMPL == 3) mv_tma2<0>(a, off, nv, dyn);
    else mv_tma2<1>(a, off, nv, dyn);
  }
}

__global__ void fill(uint16_t* p, size_t n, int seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = (uint16_t)(0x3c00 + ((i * 2654435761u + seed) & 0x3ff));  // bf16 in [1, 2)
}

int main(int argc, char** argv) {
  const size_t N = (argc > 1 ? atoll(argv[1]) : 64) << 20;
  CK(cudaSetDevice(0));
  std::vector<char*> S(kMax), Dd(kMax);
  for (int i = 0; i < kMax; i++) {
    CK(cudaMalloc(&S[i], N));
    CK(cudaMalloc(&Dd[i], N));
    fill<<<1024, 256>>>((uint16_t*)S[i], N / 2, i);
  }
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  struct Shape { int K, M; };
  const Shape shapes[] = {{5, 8}, {5, 5}, {4, 1}, {1, 3}, {1, 1}};
  struct Cfg { const char* name; int impl, U, PF, NST, SB, VPT, ctas_per_sm; };
  std::vector<Cfg> cfgs = {
      {"lgsts_u4_pf2", 1, 4, 2, 0, 0, 0, 2},     {"tma2_3x16k_c4", 3, 0, 0, 3, 16384, 4, 4},
      {"tma2_4x12k_c4", 3, 0, 0, 4, 12288, 4, 4}, {"tma2_2x24k_c4", 3, 0, 0, 2, 24576, 4, 4},
      {"s2g_3x16k_c4", 4, 0, 0, 3, 16384, 4, 4},  {"s2g_4x12k_c4", 4, 0, 0, 4, 12288, 4, 4},
      {"tma2_3x24k_c3", 3, 0, 0, 3, 24576, 4, 3}, {"s2g_3x24k_c3", 4, 0, 0, 3, 24576, 4, 3},
      {"tma2_4x24k_c2", 3, 0, 0, 4, 24576, 4, 2}, {"s2g_4x24k_c2", 4, 0, 0, 4, 24576, 4, 2},
      {"tma2_3x8k_c6", 3, 0, 0, 3, 8192, 4, 6},
  };
  const size_t blks[] = {128 << 10};
  for (const Shape& sh : shapes)
    for (size_t BLK : blks)
      for (const Cfg& c : cfgs) {
        Args a;
        memset(&a, 0, sizeof(a));
        for (int i = 0; i < sh.K; i++) a.src[i] = S[i];
        for (int i = 0; i < sh.M; i++) a.dst[i] = Dd[i];
        a.K = sh.K;
        a.M = sh.M;
        a.N = N;
        a.BLK = BLK;
        a.U = c.U;
        a.PF = c.PF;
        a.NST = c.NST;
        a.SB = c.SB;
        a.VPT = c.VPT;
        size_t smem = c.impl == 1 ? (size_t)sh.K * c.U * 128 * 16 : c.impl >= 2 ? (size_t)c.NST * c.SB : 0;
        void (*fn)(Args) = c.impl == 0   ? k_probe<0, 4>
                           : c.impl == 1 ? k_probe<1, 4>
                           : c.impl == 2 ? k_probe<2, 4>
                           : c.impl == 3 ? k_probe<3, 4>
                                         : k_probe<4, 4>;
        CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        if (c.impl >= 2 && (size_t)sh.K * 16 * 32 > (size_t)c.SB) continue;
        const int grid = 148 * c.ctas_per_sm;
        float best = 1e30f;
        for (int rep = 0; rep < 5; rep++) {
          CK(cudaEventRecord(e0));
          fn<<<grid, 128, smem>>>(a);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          CK(cudaGetLastError());
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (rep > 0 && ms < best) best = ms;
        }
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, 128, smem));
        const double traffic = (double)(sh.K + sh.M) * N;
        printf("{\"K\": %d, \"M\": %d, \"blk_kb\": %zu, \"impl\": \"%s\", \"grid\": %d, \"occ\": %d, \"ms\": %.4f, "
               "\"GBps\": %.1f}\n",
               sh.K, sh.M, BLK >> 10, c.name, grid, occ, best, traffic / (best * 1e-3) / 1e9);
        fflush(stdout);
      }
  return 0;
}
