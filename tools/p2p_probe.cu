// P2P NVLink probe: achievable push (remote st) and pull (remote ld) bandwidth
// from one GPU to 1..n-1 peers at once, and all GPUs concurrently, single process with peer access.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_probe tools/p2p_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

struct Targets { int4* p[8]; int n; };

// each CTA streams its share of `bytes` to/from each target (targets interleaved by CTA)
template <bool PUSH, int UNROLL>
__global__ void __launch_bounds__(512) xfer(int4* local, Targets t, size_t n16) {
  int tgt = blockIdx.x % t.n;
  int cta = blockIdx.x / t.n;
  int ctas = gridDim.x / t.n;
  int4* remote = t.p[tgt];
  size_t stride = (size_t)ctas * blockDim.x * UNROLL;
  for (size_t base = (size_t)cta * blockDim.x * UNROLL + threadIdx.x; base < n16; base += stride) {
    int4 v[UNROLL];
    if (PUSH) {
#pragma unroll
      for (int u = 0; u < UNROLL; u++) { size_t i = base + (size_t)u * blockDim.x; if (i < n16) v[u] = local[i]; }
#pragma unroll
      for (int u = 0; u < UNROLL; u++) { size_t i = base + (size_t)u * blockDim.x; if (i < n16) remote[i] = v[u]; }
    } else {
#pragma unroll
      for (int u = 0; u < UNROLL; u++) { size_t i = base + (size_t)u * blockDim.x; if (i < n16) v[u] = __ldcg(remote + i); }
#pragma unroll
      for (int u = 0; u < UNROLL; u++) { size_t i = base + (size_t)u * blockDim.x; if (i < n16) local[i] = v[u]; }
    }
  }
}

int main(int argc, char** argv) {
  int ndev; CK(cudaGetDeviceCount(&ndev));
  printf("{\"ndev\": %d}\n", ndev);
  for (int i = 0; i < ndev; i++) {
    cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, i));
    int mc = 0; cudaDeviceGetAttribute(&mc, (cudaDeviceAttr)132 /*cudaDevAttrMulticastSupported? probe*/, i);
    printf("dev %d %s sms=%d l2=%d MB clock=%d\n", i, pr.name, pr.multiProcessorCount, pr.l2CacheSize >> 20, pr.clockRate);
    for (int j = 0; j < ndev; j++) if (j != i) { int a; CK(cudaDeviceCanAccessPeer(&a, i, j)); printf("  peer %d->%d %d\n", i, j, a); }
  }
  if (ndev < 2) return 0;
  for (int i = 0; i < ndev; i++) { CK(cudaSetDevice(i)); for (int j = 0; j < ndev; j++) if (j != i) CK(cudaDeviceEnablePeerAccess(j, 0)); }
  const size_t bytes = 256ull << 20;  // per target
  std::vector<int4*> bufL(ndev), bufR(ndev);
  for (int i = 0; i < ndev; i++) {
    CK(cudaSetDevice(i));
    CK(cudaMalloc(&bufL[i], bytes * 8)); CK(cudaMalloc(&bufR[i], bytes * 8));
    CK(cudaMemset(bufL[i], 1, bytes * 8)); CK(cudaMemset(bufR[i], 2, bytes * 8));
  }
  size_t n16 = bytes / 16;
  int ctas_list[] = {8, 16, 32, 64, 128};
  for (int push = 1; push >= 0; push--) {
    for (int npeers = 1; npeers < ndev; npeers++) {
      for (int c : ctas_list) {
        // single sender: GPU0 -> peers 1..npeers ; all-concurrent: every GPU i -> (i+1..i+npeers)%ndev
        for (int all = 0; all < 2; all++) {
          std::vector<cudaEvent_t> e0(ndev), e1(ndev);
          int senders = all ? ndev : 1;
          float worst = 0;
          for (int rep = 0; rep < 4; rep++) {
            for (int s = 0; s < senders; s++) {
              CK(cudaSetDevice(s));
              if (rep == 0) { CK(cudaEventCreate(&e0[s])); CK(cudaEventCreate(&e1[s])); }
              Targets t; t.n = npeers;
              for (int k = 0; k < npeers; k++) t.p[k] = bufR[(s + 1 + k) % ndev] + (size_t)s * n16;  // distinct region per sender
              int grid = c * npeers;
              CK(cudaEventRecord(e0[s]));
              if (push) xfer<true, 4><<<grid, 512>>>(bufL[s], t, n16);
              else xfer<false, 4><<<grid, 512>>>(bufL[s] + 0, t, n16);
              CK(cudaEventRecord(e1[s]));
            }
            for (int s = 0; s < senders; s++) { CK(cudaSetDevice(s)); CK(cudaDeviceSynchronize()); }
            if (rep > 0) {
              float mx = 0; for (int s = 0; s < senders; s++) { float ms; CK(cudaEventElapsedTime(&ms, e0[s], e1[s])); if (ms > mx) mx = ms; }
              if (rep == 1 || mx < worst) worst = mx;
            }
          }
          double gbs = (double)bytes * npeers / (worst * 1e-3) / 1e9;
          printf("{\"mode\": \"%s\", \"all\": %d, \"npeers\": %d, \"ctas_per_peer\": %d, \"ms\": %.3f, \"GBps_per_gpu\": %.1f}\n",
                 push ? "push" : "pull", all, npeers, c, worst, gbs);
          for (int s = 0; s < senders; s++) { CK(cudaSetDevice(s)); cudaEventDestroy(e0[s]); cudaEventDestroy(e1[s]); }
        }
      }
    }
  }
  return 0;
}
