// kernels_legacy.cu — the legacy build of the pipeline kernels (namespace hetccl::k2): 2 CTAs per SM with up
// to 255 registers, fold sources staged through shared memory by cp.async (LDGSTS) instead of the TMA ring.
// Used by one-rank-per-GPU comms by default (HETCCL_LEGACY), where the movers' NVLink stores, not HBM,
// bound the time (r02t/r02y: the TMA build lost 5-20% there). Same device code as kernels.cu.
#define HETCCL_KNS k2
#define HETCCL_KERNEL_CPS 2
#define HETCCL_LEGACY_MOVERS 1
#define HETCCL_TMA 0
#include "kernels.cu"
