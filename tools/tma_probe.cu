// Copy-engine probe: per-CTA and aggregate bandwidth of the two ways a hetccl stage can move bytes,
// local HBM -> local HBM and local HBM -> peer HBM over NVLink (push) / peer -> local (pull):
//   ldst<U>: 16-B LDG/STG, U vectors in flight per thread, 512 threads per CTA
//   tma<B>:  one elected thread per CTA, cp.async.bulk global->shared (mbarrier complete_tx) then
//            cp.async.bulk shared->global (bulk_group), B buffers of CH bytes in flight
// Verifies the copied bytes. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t e = (x);                                                                          \
    if (e != cudaSuccess) {                                                                       \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);           \
      exit(1);                                                                                    \
    }                                                                                             \
  } while (0)

template <int U>
__global__ void __launch_bounds__(512) ldst(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t base = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < n16; base += stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      size_t i = base + (size_t)u * blockDim.x;
      if (i < n16) v[u] = __ldcg(src + i);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      size_t i = base + (size_t)u * blockDim.x;
      if (i < n16) dst[i] = v[u];
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// every CTA copies chunks ch = blockIdx.x, +gridDim.x, ... of CH bytes through a ring of NB smem buffers
__global__ void __launch_bounds__(32) tma_copy(const char* src, char* dst, size_t bytes, int CH, int NB) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[16];
  if (threadIdx.x != 0) return;
  for (int b = 0; b < NB; b++)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[b])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[16] = {0};
  const size_t nch = bytes / CH;
  int issued = 0;
  // software pipeline: load chunk i into buffer i%NB; when it lands, store it out
  size_t my_n = (nch > blockIdx.x) ? (nch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  for (size_t k = 0; k < my_n + NB; k++) {
    if (k < my_n) {
      int b = k % NB;
      if (k >= (size_t)NB) {
        // buffer b was last stored at k-NB; make sure its smem was read by the bulk store
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");
      }
      size_t c = blockIdx.x + k * gridDim.x;
      uint32_t s = smem_u32(sm + (size_t)b * CH), mb = smem_u32(&bar[b]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(s), "l"(src + c * CH), "r"(CH), "r"(mb) : "memory");
      issued++;
    }
    if (k >= (size_t)NB - 1 && k - (NB - 1) < my_n) {
      size_t kk = k - (NB - 1);
      int b = kk % NB;
      uint32_t mb = smem_u32(&bar[b]);
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(mb), "r"(phase[b]) : "memory");
      phase[b] ^= 1;
      size_t c = blockIdx.x + kk * gridDim.x;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CH),
                   "r"(smem_u32(sm + (size_t)b * CH)), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void fill(int4* p, size_t n16, int seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_int4((int)i ^ seed, (int)(i >> 3) + seed, seed, (int)i * 7);
}
__global__ void check(const int4* p, size_t n16, int seed, unsigned long long* bad) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    int4 v = p[i];
    if (v.x != ((int)i ^ seed) || v.y != (int)(i >> 3) + seed || v.z != seed || v.w != (int)i * 7) atomicAdd(bad, 1ull);
  }
}

int main() {
  int ndev;
  CK(cudaGetDeviceCount(&ndev));
  const size_t bytes = 512ull << 20;
  const size_t n16 = bytes / 16;
  std::vector<char*> A(ndev), B(ndev);
  for (int i = 0; i < ndev; i++) {
    CK(cudaSetDevice(i));
    for (int j = 0; j < ndev; j++)
      if (j != i) CK(cudaDeviceEnablePeerAccess(j, 0));
    CK(cudaMalloc(&A[i], bytes));
    CK(cudaMalloc(&B[i], bytes));
    CK(cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  }
  unsigned long long* bad;
  CK(cudaSetDevice(0));
  CK(cudaMallocManaged(&bad, 8));
  struct Mode { const char* name; int src_dev, dst_dev, run_dev; };
  std::vector<Mode> modes = {{"local", 0, 0, 0}};
  if (ndev > 1) {
    modes.push_back({"push", 0, 1, 0});
    modes.push_back({"pull", 1, 0, 0});
  }
  int grids[] = {16, 32, 64, 128, 148};
  for (auto& m : modes) {
    CK(cudaSetDevice(m.src_dev));
    fill<<<1024, 256>>>((int4*)A[m.src_dev], n16, 11);
    CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(m.run_dev));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int g : grids) {
      for (int impl = 0; impl < 6; impl++) {
        // 0: ldst U4, 1: ldst U8, 2: tma 4x32K, 3: tma 6x32K, 4: tma 3x64K, 5: tma 12x16K
        int CH = 32768, NB = 4;
        if (impl == 3) NB = 6;
        if (impl == 4) { CH = 65536; NB = 3; }
        if (impl == 5) { CH = 16384; NB = 12; }
        CK(cudaSetDevice(m.dst_dev));
        CK(cudaMemset(B[m.dst_dev], 0, bytes));
        CK(cudaDeviceSynchronize());
        CK(cudaSetDevice(m.run_dev));
        float best = 1e30f;
        for (int rep = 0; rep < 4; rep++) {
          CK(cudaEventRecord(e0));
          if (impl == 0) ldst<4><<<g, 512>>>((const int4*)A[m.src_dev], (int4*)B[m.dst_dev], n16);
          else if (impl == 1) ldst<8><<<g, 512>>>((const int4*)A[m.src_dev], (int4*)B[m.dst_dev], n16);
          else tma_copy<<<g, 32, (size_t)CH * NB>>>(A[m.src_dev], B[m.dst_dev], bytes, CH, NB);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          CK(cudaGetLastError());
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (rep > 0 && ms < best) best = ms;
        }
        CK(cudaSetDevice(m.dst_dev));
        *bad = 0;
        check<<<1024, 256>>>((const int4*)B[m.dst_dev], n16, 11, bad);
        CK(cudaDeviceSynchronize());
        const char* nm[] = {"ldst_u4", "ldst_u8", "tma_4x32k", "tma_6x32k", "tma_3x64k", "tma_12x16k"};
        printf("{\"mode\": \"%s\", \"impl\": \"%s\", \"ctas\": %d, \"ms\": %.4f, \"GBps\": %.1f, \"per_cta_GBps\": %.2f, "
               "\"bad\": %llu}\n",
               m.name, nm[impl], g, best, bytes / (best * 1e-3) / 1e9, bytes / (best * 1e-3) / 1e9 / g, *bad);
        fflush(stdout);
      }
    }
  }
  return 0;
}
