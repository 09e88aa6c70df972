/*
 * hetccl.h — C ABI of the B200-native hierarchical collective library (HetCCL hot path,
 * arXiv 2601.22585). Pure C; no torch or CUDA types in the signatures (a stream is passed as the
 * opaque `hetcclStream_t`, which IS a `cudaStream_t`; pass 0 for the legacy default stream).
 *
 * What the library computes (see DESIGN.md §1-3 for the full readings):
 *   All-Reduce, Reduce-Scatter, All-Gather and Broadcast over n ranks split into D "device
 *   domains" (the paper's vendor groups). The paper evaluates exactly these collectives
 *   (§5.2 "All-Reduce, All-Gather, Reduce-Scatter, Reduce, Broadcast, and
 *   All-to-All"; App. E.1) and composes them from vendor-local collectives plus a
 *   cross-vendor layer (§4 "Key Approach"; §4.2). The composition it
 *   leaves open is read as SPEC.md:350 / SPEC.md:404: intra-domain reduce-scatter -> cross-domain
 *   exchange of partials -> intra-domain all-gather. Signatures, in-place rules and enum VALUES copy
 *   NCCL's, because the paper's boundary is "intercepting and overriding NCCL or RCCL symbols"
 *   (§4.4).
 *
 * Floating-point order (reading R3): for every element, ascending rank within each
 * domain, then ascending domain id; 16-bit types accumulate in fp32 and are rounded (RNE) once at
 * the domain boundary and once at the end (reading R6). int32 sums wrap mod 2^32 (reading R8).
 * Results are deterministic and identical on every rank.
 *
 * Ownership: the caller owns send/recv buffers and streams; buffers are device memory of the
 * comm's device, must stay untouched until the stream passes the op, and need no registration.
 * The library owns the comm, its scratch ring, flags and peer mappings until hetccl_comm_destroy.
 *
 * Ordering: every op is enqueued on `stream` and returns without a host sync. Every rank must issue
 * the same ops in the same order with the same count/dtype/op/root (as in NCCL; a mismatch is
 * undefined and not detected). One comm must not run two ops concurrently (use one comm per
 * concurrent stream). A device-side spin timeout (HETCCL_TIMEOUT_S, default 30 s) ends a stuck
 * op early; hetccl_comm_get_async_error then reports it.
 *
 * Errors are return codes only (no exceptions or abort across the ABI); the detail text of the
 * last failure on a comm is available from hetccl_get_last_error.
 */
#ifndef HETCCL_H
#define HETCCL_H

#include <stddef.h>

#if defined(__GNUC__)
#define HETCCL_API __attribute__((visibility("default")))
#else
#define HETCCL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define HETCCL_VERSION 100 /* 0.1.0 */
#define HETCCL_MAX_RANKS 16
#define HETCCL_BLOB_BYTES 512 /* bytes per rank written by hetccl_comm_export */

typedef struct hetcclComm* hetcclComm_t;
struct CUstream_st;
typedef struct CUstream_st* hetcclStream_t; /* == cudaStream_t */

typedef enum {
  hetcclSuccess = 0,
  hetcclUnhandledCudaError = 1, /* a CUDA runtime call failed */
  hetcclSystemError = 2,        /* IPC import / host allocation failed */
  hetcclInternalError = 3,      /* device-side timeout or protocol failure */
  hetcclInvalidArgument = 4,    /* null pointer, bad map/dtype/op/root/count, illegal overlap */
  hetcclInvalidUsage = 5        /* comm not connected, wrong device, wrong comm kind */
} hetcclResult_t;

typedef enum { hetcclInt32 = 2, hetcclFloat16 = 6, hetcclFloat32 = 7, hetcclBfloat16 = 9 } hetcclDataType_t;
typedef enum { hetcclSum = 0, hetcclMax = 2, hetcclMin = 3 } hetcclRedOp_t;

/* ---------------------------------------------------------------- communicators ------------- */

/* Library version (HETCCL_VERSION). */
HETCCL_API hetcclResult_t hetccl_get_version(int* version);

/*
 * Map validation only (no CUDA): rank_to_domain[r] in [0, D) for r in [0, nranks), ids dense
 * (every id 0..D-1 used), 1 <= nranks <= HETCCL_MAX_RANKS. Writes D to *ndomains if non-null.
 * Returns hetcclInvalidArgument otherwise.
 */
HETCCL_API hetcclResult_t hetccl_validate_map(int nranks, const int* rank_to_domain, int* ndomains);

/*
 * One process per GPU, two-phase bootstrap:
 *   hetccl_comm_init   allocates this rank's symmetric scratch ring + flags on `cuda_device`
 *                      (the map is copied; identical on all ranks);
 *   hetccl_comm_export writes this rank's HETCCL_BLOB_BYTES-byte blob (CUDA IPC handles) to `blob`
 *                      (*blob_bytes in: capacity, out: bytes written);
 *   the caller all-gathers the blobs (e.g. torch.distributed.all_gather_object over gloo), then
 *   hetccl_comm_connect takes nranks blobs concatenated in rank order (blob_bytes = nranks *
 *                      HETCCL_BLOB_BYTES), opens the peers' memory and checks that every rank
 *                      passed the same map and geometry (hetcclInvalidUsage if not).
 */
HETCCL_API hetcclResult_t hetccl_comm_init(hetcclComm_t* comm, int nranks, int rank, const int* rank_to_domain,
                                int cuda_device);
HETCCL_API hetcclResult_t hetccl_comm_export(hetcclComm_t comm, void* blob, size_t* blob_bytes);
HETCCL_API hetcclResult_t hetccl_comm_connect(hetcclComm_t comm, const void* blobs, size_t blob_bytes);

/* Single process driving ndev GPUs (tests, bench): comms[i] is rank i on device devlist[i];
 * peer access is enabled between all pairs. Ops are then issued per comm (any order of launch). */
HETCCL_API hetcclResult_t hetccl_comm_init_all(hetcclComm_t* comms, int ndev, const int* devlist, const int* rank_to_domain);

/*
 * Rank-multiplexed comm: all `nranks` logical ranks live on ONE device and every op runs as ONE
 * cooperative kernel over all ranks' buffers (rank = blockIdx.y). Same device code and protocol as
 * the multi-GPU path; used to check 8-rank splits on fewer GPUs and for the 1-GPU
 * bench. Use the hetccl_mux_* entry points with per-rank buffer arrays.
 */
HETCCL_API hetcclResult_t hetccl_comm_init_mux(hetcclComm_t* comm, int nranks, const int* rank_to_domain, int cuda_device);

/* Frees scratch, flags and peer mappings. Synchronizes the comm's device first. */
HETCCL_API hetcclResult_t hetccl_comm_destroy(hetcclComm_t comm);

/* Rank, size, domain of this rank, number of domains, index within its domain, domain size. */
HETCCL_API hetcclResult_t hetccl_comm_info(hetcclComm_t comm, int* rank, int* nranks, int* domain, int* ndomains,
                                int* domain_rank, int* domain_size);

/*
 * NVLS mode (opt-in). With HETCCL_NVLS=1 in the environment of
 * hetccl_comm_init_all or of every rank's hetccl_comm_init (one rank per process: the domain leader hands its
 * multicast handle to the members through a unix socket during hetccl_comm_connect, and the ranks agree before
 * switching), and every domain of the same size d >= 2 on devices with multicast support,
 * each domain gets an NVLink SHARP multicast object and hetccl_allreduce (bf16/fp16/fp32 sum, 16-byte
 * aligned buffers) runs its intra-domain reduce-scatter inside the switch (multimem.ld_reduce) and its
 * intra-domain all-gather as one multicast store (multimem.st); the cross-domain exchange and fold stay
 * P2P in ascending domain order. 16-bit inputs are staged in fp32 (HETCCL_NVLS_WIDE=1, the default: the
 * switch's fp32 adds are round-to-nearest-even, its 16-bit ones are not) and each partial is narrowed
 * once, so results meet the R7 gate (elementwise 1e-2 * sum|x|, normwise 1e-2); the switch's summation
 * order is not R3's, so they are not bitwise those of the oracle (R21). Other dtypes, ops and
 * unaligned buffers keep the P2P path.
 *   enabled : 1 if this comm runs All-Reduce in NVLS mode, else 0 (hetccl_get_last_error says why).
 *   buffer  : this rank's view of its multicast-bound buffer (device memory owned by the comm, valid
 *             until hetccl_comm_destroy), or NULL. An in-place f32 All-Reduce on it (sendbuf == recvbuf ==
 *             buffer, count * size a multiple of 16 bytes, at most *bytes) skips the copies in and out;
 *             a 16-bit All-Reduce whose buffers overlap it is hetcclInvalidArgument while staging wide
 *             (the buffer holds the fp32 staging copy).
 *   bytes   : the buffer's usable size (the chunk size, HETCCL_NVLS_MB rounded to the multicast
 *             granularity), or 0.
 * Any output pointer may be NULL. hetcclInvalidArgument on a null comm.
 */
HETCCL_API hetcclResult_t hetccl_comm_nvls(hetcclComm_t comm, int* enabled, void** buffer, size_t* bytes);

/* hetcclInternalError if a device-side timeout was recorded on this comm since init (sticky). */
HETCCL_API hetcclResult_t hetccl_comm_get_async_error(hetcclComm_t comm);

HETCCL_API const char* hetccl_get_error_string(hetcclResult_t r);
HETCCL_API const char* hetccl_get_last_error(hetcclComm_t comm); /* detail of the last non-success on comm */

/* ----------------------------------------------------------------- collectives ------------- */
/*
 * All pointers are device pointers on the comm's device. count == 0 is a successful no-op.
 *
 * hetccl_allreduce: recvbuf[i] = reduction over all ranks of sendbuf[i], i < count; identical on
 *   every rank. In place iff sendbuf == recvbuf.
 * hetccl_reduce_scatter: sendbuf holds nranks*recvcount elements; rank r receives block r of the
 *   reduction. In place iff recvbuf == sendbuf + rank*recvcount (elements).
 * hetccl_all_gather: recvbuf holds nranks*sendcount elements; block j is rank j's sendbuf.
 *   In place iff sendbuf == recvbuf + rank*sendcount.
 * hetccl_broadcast: every rank's recvbuf = root's sendbuf (count elements); sendbuf is read on the
 *   root only (may be NULL elsewhere). In place iff sendbuf == recvbuf.
 * hetccl_reduce (App. E.1 "Reduce"): the root's recvbuf = the
 *   All-Reduce result (same order and rounding); recvbuf is written on the root only (may be NULL
 *   elsewhere). In place iff sendbuf == recvbuf.
 * hetccl_all_to_all (App. E.1 "All-to-All"): sendbuf and recvbuf hold nranks blocks of
 *   `count` elements; block j of sendbuf goes to rank j, block j of recvbuf comes from rank j. Send and
 *   recv must not overlap.
 * Any other overlap of send and recv ranges is hetcclInvalidArgument.
 */
HETCCL_API hetcclResult_t hetccl_allreduce(const void* sendbuf, void* recvbuf, size_t count, hetcclDataType_t dt,
                                hetcclRedOp_t op, hetcclComm_t comm, hetcclStream_t stream);
HETCCL_API hetcclResult_t hetccl_reduce_scatter(const void* sendbuf, void* recvbuf, size_t recvcount, hetcclDataType_t dt,
                                     hetcclRedOp_t op, hetcclComm_t comm, hetcclStream_t stream);
HETCCL_API hetcclResult_t hetccl_all_gather(const void* sendbuf, void* recvbuf, size_t sendcount, hetcclDataType_t dt,
                                 hetcclComm_t comm, hetcclStream_t stream);
HETCCL_API hetcclResult_t hetccl_broadcast(const void* sendbuf, void* recvbuf, size_t count, hetcclDataType_t dt, int root,
                                hetcclComm_t comm, hetcclStream_t stream);
HETCCL_API hetcclResult_t hetccl_reduce(const void* sendbuf, void* recvbuf, size_t count, hetcclDataType_t dt,
                                        hetcclRedOp_t op, int root, hetcclComm_t comm, hetcclStream_t stream);
HETCCL_API hetcclResult_t hetccl_all_to_all(const void* sendbuf, void* recvbuf, size_t count, hetcclDataType_t dt,
                                            hetcclComm_t comm, hetcclStream_t stream);

/* Rank-multiplexed variants: sendbufs[r] / recvbufs[r] for every logical rank r of a mux comm. */
HETCCL_API hetcclResult_t hetccl_mux_allreduce(const void* const* sendbufs, void* const* recvbufs, size_t count,
                                    hetcclDataType_t dt, hetcclRedOp_t op, hetcclComm_t comm, hetcclStream_t stream);
HETCCL_API hetcclResult_t hetccl_mux_reduce_scatter(const void* const* sendbufs, void* const* recvbufs, size_t recvcount,
                                         hetcclDataType_t dt, hetcclRedOp_t op, hetcclComm_t comm,
                                         hetcclStream_t stream);
HETCCL_API hetcclResult_t hetccl_mux_all_gather(const void* const* sendbufs, void* const* recvbufs, size_t sendcount,
                                     hetcclDataType_t dt, hetcclComm_t comm, hetcclStream_t stream);
HETCCL_API hetcclResult_t hetccl_mux_broadcast(const void* const* sendbufs, void* const* recvbufs, size_t count,
                                    hetcclDataType_t dt, int root, hetcclComm_t comm, hetcclStream_t stream);
HETCCL_API hetcclResult_t hetccl_mux_reduce(const void* const* sendbufs, void* const* recvbufs, size_t count,
                                            hetcclDataType_t dt, hetcclRedOp_t op, int root, hetcclComm_t comm,
                                            hetcclStream_t stream);
HETCCL_API hetcclResult_t hetccl_mux_all_to_all(const void* const* sendbufs, void* const* recvbufs, size_t count,
                                                hetcclDataType_t dt, hetcclComm_t comm, hetcclStream_t stream);

/* ------------------------------------------------------------- plan introspection ----------- */
/*
 * Host-only (no CUDA): the per-rank algorithmic NVLink bytes one op moves, from the same plan the
 * kernels execute. op: 0 allreduce, 1 reduce_scatter, 2 all_gather, 3 broadcast,
 * 4 reduce, 5 all_to_all (count = elements per block).
 * count = the op's `count` argument (recvcount / sendcount for RS / AG). Writes bytes sent and
 * received by `rank` over the peer fabric, and the tile geometry (elements per tile, tiles,
 * channels) the pipelined launch would use with `nchannels` channels (0 = a one-rank-per-GPU comm's
 * default under the current environment, including the mid-size All-Reduce channel cap; sizes that
 * take the one-shot All-Reduce below its cutoff are reported as if pipelined).
 */
typedef struct {
  size_t bytes_sent;
  size_t bytes_recv;
  size_t tile_elems;
  size_t ntiles;
  int nchannels;
  int nslots;
} hetcclPlanInfo_t;
HETCCL_API hetcclResult_t hetccl_plan_info(int nranks, const int* rank_to_domain, int rank, int op, size_t count,
                                hetcclDataType_t dt, int root, int nchannels, hetcclPlanInfo_t* info);

/*
 * Host-only (no CUDA): the pipeline schedule `rank` runs for one op. Logical stage s
 * (0..nstages-1) is active iff bit s of `active` is set (identical on every rank). Before stage s of
 * a tile, every sender in wait_mask[s] must have signalled counter wait_ctr[s] (0 S1, 1 S2, 2 AG,
 * 3 S3; 7 = none) for that tile; after it, counter sig_ctr[s] of every rank in sig_mask[s] is
 * signalled. `writes` = ranks whose scratch this rank writes. For tests of the protocol's symmetry.
 */
typedef struct {
  int nstages;
  unsigned int active;
  int wait_ctr[8];
  unsigned int wait_mask[8];
  int sig_ctr[8];
  unsigned int sig_mask[8];
  unsigned int writes;
} hetcclStagePlan_t;
HETCCL_API hetcclResult_t hetccl_plan_stages(int nranks, const int* rank_to_domain, int rank, int op, int root,
                                             hetcclStagePlan_t* plan);

/*
 * Symmetric recv buffers (SURVEY NEXT-4 "user-buffer registration for zero-copy"). Every rank allocates
 * a buffer of the same size with hetccl_mem_alloc (device memory of the comm's device, owned by the
 * comm until hetccl_mem_free / hetccl_comm_destroy), exports it (HETCCL_BLOB_BYTES per rank), the caller
 * all-gathers the blobs and passes them, concatenated in rank order, to hetccl_mem_connect. From then
 * on an All-Reduce whose recvbuf lies inside such a buffer is taken to use the SAME offset in every
 * rank's buffer (the caller's contract), and final results are written straight into the peers'
 * buffers instead of being staged through scratch. Rank-multiplexed comms need no registration.
 * HETCCL_DIRECT=0 disables the direct path.
 */
HETCCL_API hetcclResult_t hetccl_mem_alloc(hetcclComm_t comm, size_t bytes, void** ptr);
HETCCL_API hetcclResult_t hetccl_mem_export(hetcclComm_t comm, void* ptr, void* blob, size_t* blob_bytes);
HETCCL_API hetcclResult_t hetccl_mem_connect(hetcclComm_t comm, void* ptr, const void* blobs, size_t blob_bytes);
HETCCL_API hetcclResult_t hetccl_mem_free(hetcclComm_t comm, void* ptr);

/*
 * Profiling aid. With HETCCL_TRACE_ITERS=K set when the comm is created, every op records, per
 * (local rank, channel) CTA and pipeline iteration it < K, eight globaltimer stamps in ns: wait start,
 * work start (all waits satisfied), work end, release fence done, and the end of logical stages 0..3 as
 * seen by thread 0 (0 if the stage did not run). This copies the LAST op's stamps to
 * `host` as uint64 [shape0 local ranks][shape1 channels][shape2 = K iterations][8] (synchronizes
 * the device; unused iterations are 0). shape[0..2] are written; all zero if tracing is off. With
 * host == NULL only the shape is written.
 */
HETCCL_API hetcclResult_t hetccl_comm_get_trace(hetcclComm_t comm, void* host, size_t bytes, int* shape);

#ifdef __cplusplus
}
#endif
#endif /* HETCCL_H */
