"""Python binding of libhetccl.so (include/hetccl.h) — argument marshalling only.

Every collective runs in the library's sm_100a kernels; this module converts torch tensors / ints
to pointers and sizes, raises on a non-success return code, and offers a torch.distributed
bootstrap for the one-process-per-GPU mode (the blob exchange of SURVEY §3.2). There is no CPU
fallback: importing a collective without the built extension raises.

Function names follow the C ABI (``hetccl_allreduce`` ...); ``allreduce`` etc. are the same calls
taking tensors.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# HETCCL_LIB selects an in-tree build variant (A/B experiments); default libhetccl.so
_LIB_PATH = os.path.join(_HERE, os.environ.get("HETCCL_LIB", "libhetccl.so"))

INT32, FLOAT16, FLOAT32, BFLOAT16 = 2, 6, 7, 9
SUM, MAX, MIN = 0, 2, 3
OP_ALLREDUCE, OP_REDUCE_SCATTER, OP_ALL_GATHER, OP_BROADCAST, OP_REDUCE, OP_ALL_TO_ALL = 0, 1, 2, 3, 4, 5
BLOB_BYTES = 512
MAX_RANKS = 16
_RESULT = {0: "hetcclSuccess", 1: "hetcclUnhandledCudaError", 2: "hetcclSystemError", 3: "hetcclInternalError",
           4: "hetcclInvalidArgument", 5: "hetcclInvalidUsage"}
_OPS = {"sum": SUM, "max": MAX, "min": MIN}


class HetcclError(RuntimeError):
    def __init__(self, code, detail=""):
        self.code = code
        super().__init__(f"{_RESULT.get(code, code)}: {detail}")


class StagePlan(ctypes.Structure):
    _fields_ = [("nstages", ctypes.c_int), ("active", ctypes.c_uint), ("wait_ctr", ctypes.c_int * 8),
                ("wait_mask", ctypes.c_uint * 8), ("sig_ctr", ctypes.c_int * 8), ("sig_mask", ctypes.c_uint * 8),
                ("writes", ctypes.c_uint)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("bytes_sent", ctypes.c_size_t), ("bytes_recv", ctypes.c_size_t), ("tile_elems", ctypes.c_size_t),
                ("ntiles", ctypes.c_size_t), ("nchannels", ctypes.c_int), ("nslots", ctypes.c_int)]


EXPORTED = [
    "hetccl_get_version", "hetccl_validate_map", "hetccl_comm_init", "hetccl_comm_export", "hetccl_comm_connect",
    "hetccl_comm_init_all", "hetccl_comm_init_mux", "hetccl_comm_destroy", "hetccl_comm_info",
    "hetccl_comm_get_async_error", "hetccl_get_error_string", "hetccl_get_last_error", "hetccl_allreduce",
    "hetccl_reduce_scatter", "hetccl_all_gather", "hetccl_broadcast", "hetccl_mux_allreduce",
    "hetccl_mux_reduce_scatter", "hetccl_mux_all_gather", "hetccl_mux_broadcast", "hetccl_plan_info",
    "hetccl_plan_stages", "hetccl_comm_get_trace", "hetccl_reduce", "hetccl_all_to_all", "hetccl_mux_reduce",
    "hetccl_mux_all_to_all", "hetccl_mem_alloc", "hetccl_mem_export", "hetccl_mem_connect", "hetccl_mem_free",
    "hetccl_comm_nvls",
]

_lib = None


def lib():
    """Load libhetccl.so (built in-tree by build.py / __graft_entry__.build()). Raises if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: build it with `python -m paper_2601_22585_b200.build`")
    L = ctypes.CDLL(_LIB_PATH)
    c_int, c_size, vp, pp = ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)
    ip = ctypes.POINTER(ctypes.c_int)
    sig = {
        "hetccl_get_version": [ip],
        "hetccl_validate_map": [c_int, ip, ip],
        "hetccl_comm_init": [pp, c_int, c_int, ip, c_int],
        "hetccl_comm_export": [vp, vp, ctypes.POINTER(c_size)],
        "hetccl_comm_connect": [vp, vp, c_size],
        "hetccl_comm_init_all": [pp, c_int, ip, ip],
        "hetccl_comm_init_mux": [pp, c_int, ip, c_int],
        "hetccl_comm_destroy": [vp],
        "hetccl_comm_info": [vp, ip, ip, ip, ip, ip, ip],
        "hetccl_comm_get_async_error": [vp],
        "hetccl_allreduce": [vp, vp, c_size, c_int, c_int, vp, vp],
        "hetccl_reduce_scatter": [vp, vp, c_size, c_int, c_int, vp, vp],
        "hetccl_all_gather": [vp, vp, c_size, c_int, vp, vp],
        "hetccl_broadcast": [vp, vp, c_size, c_int, c_int, vp, vp],
        "hetccl_reduce": [vp, vp, c_size, c_int, c_int, c_int, vp, vp],
        "hetccl_all_to_all": [vp, vp, c_size, c_int, vp, vp],
        "hetccl_mux_reduce": [pp, pp, c_size, c_int, c_int, c_int, vp, vp],
        "hetccl_mux_all_to_all": [pp, pp, c_size, c_int, vp, vp],
        "hetccl_mux_allreduce": [pp, pp, c_size, c_int, c_int, vp, vp],
        "hetccl_mux_reduce_scatter": [pp, pp, c_size, c_int, c_int, vp, vp],
        "hetccl_mux_all_gather": [pp, pp, c_size, c_int, vp, vp],
        "hetccl_mux_broadcast": [pp, pp, c_size, c_int, c_int, vp, vp],
        "hetccl_plan_info": [c_int, ip, c_int, c_int, c_size, c_int, c_int, c_int, ctypes.POINTER(PlanInfo)],
        "hetccl_plan_stages": [c_int, ip, c_int, c_int, c_int, ctypes.POINTER(StagePlan)],
        "hetccl_comm_get_trace": [vp, vp, c_size, ip],
        "hetccl_mem_alloc": [vp, c_size, pp],
        "hetccl_mem_export": [vp, vp, vp, ctypes.POINTER(c_size)],
        "hetccl_mem_connect": [vp, vp, vp, c_size],
        "hetccl_mem_free": [vp, vp],
        "hetccl_comm_nvls": [vp, ip, pp, ctypes.POINTER(c_size)],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = c_int
    L.hetccl_get_error_string.argtypes = [c_int]
    L.hetccl_get_error_string.restype = ctypes.c_char_p
    L.hetccl_get_last_error.argtypes = [vp]
    L.hetccl_get_last_error.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(rc, comm=None):
    if rc != 0:
        detail = ""
        if comm is not None:
            detail = (lib().hetccl_get_last_error(comm) or b"").decode()
        raise HetcclError(rc, detail or lib().hetccl_get_error_string(rc).decode())


def _imap(seq):
    return (ctypes.c_int * len(seq))(*[int(v) for v in seq])


# ------------------------------------------------------------------------------ dtype mapping
def dtype_code(dt):
    import torch
    m = {torch.int32: INT32, torch.float16: FLOAT16, torch.float32: FLOAT32, torch.bfloat16: BFLOAT16}
    if dt not in m:
        raise HetcclError(4, f"unsupported dtype {dt}")
    return m[dt]


def _op(op):
    return _OPS[op] if isinstance(op, str) else int(op)


def _stream(stream, like=None):
    """A raw cudaStream_t: `stream` as given, else the current stream of the device `like` (a tensor) lives on
    (a comm on another GPU than the current one must not be handed the current device's stream)."""
    if stream is None:
        import torch
        dev = like.device if like is not None and hasattr(like, "device") else None
        if dev is not None and dev.type != "cuda":
            dev = None  # a host tensor: the library rejects it (hetcclInvalidUsage); any stream will do
        return torch.cuda.current_stream(dev).cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _ptr(t):
    return None if t is None else (t if isinstance(t, int) else t.data_ptr())


# ------------------------------------------------------------------------------ communicators
def hetccl_validate_map(rank_to_domain):
    nd = ctypes.c_int(0)
    _check(lib().hetccl_validate_map(len(rank_to_domain), _imap(rank_to_domain), ctypes.byref(nd)))
    return nd.value


def hetccl_comm_init(nranks, rank, rank_to_domain, device):
    c = ctypes.c_void_p()
    _check(lib().hetccl_comm_init(ctypes.byref(c), nranks, rank, _imap(rank_to_domain), device))
    return c


def hetccl_comm_export(comm):
    buf = ctypes.create_string_buffer(BLOB_BYTES)
    n = ctypes.c_size_t(BLOB_BYTES)
    _check(lib().hetccl_comm_export(comm, buf, ctypes.byref(n)), comm)
    return buf.raw[: n.value]


def hetccl_comm_connect(comm, blobs):
    data = b"".join(blobs) if isinstance(blobs, (list, tuple)) else blobs
    _check(lib().hetccl_comm_connect(comm, data, len(data)), comm)


def hetccl_comm_init_all(devlist, rank_to_domain):
    n = len(devlist)
    arr = (ctypes.c_void_p * n)()
    _check(lib().hetccl_comm_init_all(arr, n, _imap(devlist), _imap(rank_to_domain)))
    return [ctypes.c_void_p(arr[i]) for i in range(n)]


def hetccl_comm_init_mux(nranks, rank_to_domain, device):
    c = ctypes.c_void_p()
    _check(lib().hetccl_comm_init_mux(ctypes.byref(c), nranks, _imap(rank_to_domain), device))
    return c


def hetccl_comm_destroy(comm):
    _check(lib().hetccl_comm_destroy(comm))


def hetccl_comm_info(comm):
    v = [ctypes.c_int(0) for _ in range(6)]
    _check(lib().hetccl_comm_info(comm, *[ctypes.byref(x) for x in v]), comm)
    keys = ("rank", "nranks", "domain", "ndomains", "domain_rank", "domain_size")
    return dict(zip(keys, [x.value for x in v]))


def hetccl_comm_get_async_error(comm):
    _check(lib().hetccl_comm_get_async_error(comm), comm)


def hetccl_comm_nvls(comm):
    """NVLS mode of a hetccl_comm_init_all comm (HETCCL_NVLS=1): (enabled, buffer pointer, usable bytes)."""
    on, p, nb = ctypes.c_int(0), ctypes.c_void_p(), ctypes.c_size_t(0)
    _check(lib().hetccl_comm_nvls(comm, ctypes.byref(on), ctypes.byref(p), ctypes.byref(nb)), comm)
    return bool(on.value), p.value, nb.value


def nvls_buffer(comm, numel, dtype, device):
    """Torch view (on `device`, the comm's GPU) of the first `numel` elements of the comm's multicast-bound
    buffer: an in-place All-Reduce on it skips the copies in and out of NVLS mode. Owned by the comm."""
    import torch
    on, p, nb = hetccl_comm_nvls(comm)
    es = torch.empty((), dtype=dtype).element_size()
    if not on or numel * es > nb:
        raise HetcclError(3, f"NVLS buffer unavailable or too small ({nb} bytes)")
    name = str(dtype).replace("torch.", "")
    t = torch.as_tensor(_CudaArray(p, (numel,), _TYPESTR[name] if name != "bfloat16" else "<i2"), device=f"cuda:{device}")
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


def hetccl_comm_get_trace(comm):
    """Per-iteration timestamps of the last op (HETCCL_TRACE_ITERS at comm creation): numpy uint64
    array [local ranks, channels, iterations, 10] (wait start, work start, work end, fenced, end of logical
    stages 0..3 on thread 0 — 0 where the stage did not run; iteration 0 also holds the kernel entry and exit
    stamps in words 8 and 9), or None."""
    import numpy as np
    shape = (ctypes.c_int * 3)()
    _check(lib().hetccl_comm_get_trace(comm, None, 0, shape), comm)
    if shape[0] == 0:
        return None
    out = np.zeros((shape[0], shape[1], shape[2], 10), np.uint64)
    _check(lib().hetccl_comm_get_trace(comm, out.ctypes.data, out.nbytes, shape), comm)
    return out


def hetccl_plan_info(rank_to_domain, rank, op, count, dtype=BFLOAT16, root=0, nchannels=0):
    info = PlanInfo()
    _check(lib().hetccl_plan_info(len(rank_to_domain), _imap(rank_to_domain), rank, op, count, dtype, root,
                                  nchannels, ctypes.byref(info)))
    return {f: getattr(info, f) for f, _ in PlanInfo._fields_}


def hetccl_plan_stages(rank_to_domain, rank, op, root=0):
    """The pipeline schedule of `rank` for op (host-only): dict of nstages, active, and per logical
    stage wait_ctr / wait_mask / sig_ctr / sig_mask lists, plus writes."""
    p = StagePlan()
    _check(lib().hetccl_plan_stages(len(rank_to_domain), _imap(rank_to_domain), rank, op, root, ctypes.byref(p)))
    n = p.nstages
    return {"nstages": n, "active": p.active, "wait_ctr": list(p.wait_ctr)[:n], "wait_mask": list(p.wait_mask)[:n],
            "sig_ctr": list(p.sig_ctr)[:n], "sig_mask": list(p.sig_mask)[:n], "writes": p.writes}


def init_process_group_comm(rank_to_domain, rank=None, world_size=None, device=None, group=None):
    """One process per GPU: init this rank's comm, all-gather the IPC blobs over torch.distributed
    (object collective on `group`), connect. Returns the comm handle."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group) if rank is None else rank
    world_size = dist.get_world_size(group) if world_size is None else world_size
    device = torch.cuda.current_device() if device is None else device
    comm = hetccl_comm_init(world_size, rank, rank_to_domain, device)
    blob = hetccl_comm_export(comm)
    blobs = [None] * world_size
    dist.all_gather_object(blobs, blob, group=group)
    hetccl_comm_connect(comm, blobs)
    return comm


# ------------------------------------------------------------------------------ symmetric buffers
class _CudaArray:
    """__cuda_array_interface__ view of library-owned device memory (no copy)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


_TYPESTR = {"float32": "<f4", "float16": "<f2", "int32": "<i4", "bfloat16": "<f2"}


def symmetric_empty(comm, numel, dtype, group=None):
    """Allocate `numel` elements of `dtype` as a symmetric buffer on every rank (collective over `group`,
    a gloo group works) and connect the peers' copies. Returns a torch tensor viewing the buffer; All-
    Reduces whose output lies inside it at the same offset on every rank write results straight into the
    peers' buffers. Free with hetccl_mem_free(comm, t.data_ptr()) or by destroying the comm."""
    import torch
    import torch.distributed as dist
    es = torch.empty((), dtype=dtype).element_size()
    p = ctypes.c_void_p()
    _check(lib().hetccl_mem_alloc(comm, numel * es, ctypes.byref(p)), comm)
    buf = ctypes.create_string_buffer(BLOB_BYTES)
    nb = ctypes.c_size_t(BLOB_BYTES)
    _check(lib().hetccl_mem_export(comm, p, buf, ctypes.byref(nb)), comm)
    blobs = [None] * dist.get_world_size(group)
    dist.all_gather_object(blobs, buf.raw[: nb.value], group=group)
    data = b"".join(blobs)
    _check(lib().hetccl_mem_connect(comm, p, data, len(data)), comm)
    name = str(dtype).replace("torch.", "")
    t = torch.as_tensor(_CudaArray(p.value, (numel,), _TYPESTR[name] if name != "bfloat16" else "<i2"),
                        device="cuda")
    if dtype == torch.bfloat16:
        t = t.view(torch.bfloat16)
    return t


def symmetric_empty_all(comms, numel, dtype):
    """hetccl_comm_init_all comms (one process, n GPUs): a symmetric buffer per device, connected."""
    import torch
    es = torch.empty((), dtype=dtype).element_size()
    ptrs, blobs = [], []
    for c in comms:
        p = ctypes.c_void_p()
        _check(lib().hetccl_mem_alloc(c, numel * es, ctypes.byref(p)), c)
        buf = ctypes.create_string_buffer(BLOB_BYTES)
        nb = ctypes.c_size_t(BLOB_BYTES)
        _check(lib().hetccl_mem_export(c, p, buf, ctypes.byref(nb)), c)
        ptrs.append(p)
        blobs.append(buf.raw[: nb.value])
    data = b"".join(blobs)
    out = []
    for i, (c, p) in enumerate(zip(comms, ptrs)):
        _check(lib().hetccl_mem_connect(c, p, data, len(data)), c)
        name = str(dtype).replace("torch.", "")
        t = torch.as_tensor(_CudaArray(p.value, (numel,), _TYPESTR[name] if name != "bfloat16" else "<i2"),
                            device=f"cuda:{i}")
        out.append(t.view(torch.bfloat16) if dtype == torch.bfloat16 else t)
    return out


# ------------------------------------------------------------------------------ collectives
def hetccl_allreduce(sendbuf, recvbuf, count, dtype, op, comm, stream):
    _check(lib().hetccl_allreduce(sendbuf, recvbuf, count, dtype, _op(op), comm, stream), comm)


def hetccl_reduce_scatter(sendbuf, recvbuf, recvcount, dtype, op, comm, stream):
    _check(lib().hetccl_reduce_scatter(sendbuf, recvbuf, recvcount, dtype, _op(op), comm, stream), comm)


def hetccl_all_gather(sendbuf, recvbuf, sendcount, dtype, comm, stream):
    _check(lib().hetccl_all_gather(sendbuf, recvbuf, sendcount, dtype, comm, stream), comm)


def hetccl_broadcast(sendbuf, recvbuf, count, dtype, root, comm, stream):
    _check(lib().hetccl_broadcast(sendbuf, recvbuf, count, dtype, root, comm, stream), comm)


def hetccl_reduce(sendbuf, recvbuf, count, dtype, op, root, comm, stream):
    _check(lib().hetccl_reduce(sendbuf, recvbuf, count, dtype, _op(op), root, comm, stream), comm)


def hetccl_all_to_all(sendbuf, recvbuf, count, dtype, comm, stream):
    _check(lib().hetccl_all_to_all(sendbuf, recvbuf, count, dtype, comm, stream), comm)


def _parr(xs):
    return (ctypes.c_void_p * len(xs))(*[_ptr(x) for x in xs])


def hetccl_mux_allreduce(sendbufs, recvbufs, count, dtype, op, comm, stream):
    _check(lib().hetccl_mux_allreduce(_parr(sendbufs), _parr(recvbufs), count, dtype, _op(op), comm, stream), comm)


def hetccl_mux_reduce_scatter(sendbufs, recvbufs, recvcount, dtype, op, comm, stream):
    _check(lib().hetccl_mux_reduce_scatter(_parr(sendbufs), _parr(recvbufs), recvcount, dtype, _op(op), comm, stream),
           comm)


def hetccl_mux_all_gather(sendbufs, recvbufs, sendcount, dtype, comm, stream):
    _check(lib().hetccl_mux_all_gather(_parr(sendbufs), _parr(recvbufs), sendcount, dtype, comm, stream), comm)


def hetccl_mux_broadcast(sendbufs, recvbufs, count, dtype, root, comm, stream):
    _check(lib().hetccl_mux_broadcast(_parr(sendbufs), _parr(recvbufs), count, dtype, root, comm, stream), comm)


def hetccl_mux_reduce(sendbufs, recvbufs, count, dtype, op, root, comm, stream):
    _check(lib().hetccl_mux_reduce(_parr(sendbufs), _parr(recvbufs), count, dtype, _op(op), root, comm, stream), comm)


def hetccl_mux_all_to_all(sendbufs, recvbufs, count, dtype, comm, stream):
    _check(lib().hetccl_mux_all_to_all(_parr(sendbufs), _parr(recvbufs), count, dtype, comm, stream), comm)


# tensor conveniences (same calls; count/dtype taken from the tensors)
def allreduce(send, recv, comm, op="sum", stream=None):
    hetccl_allreduce(_ptr(send), _ptr(recv), recv.numel(), dtype_code(recv.dtype), op, comm, _stream(stream, recv))


def reduce_scatter(send, recv, comm, op="sum", stream=None):
    hetccl_reduce_scatter(_ptr(send), _ptr(recv), recv.numel(), dtype_code(recv.dtype), op, comm, _stream(stream, recv))


def all_gather(send, recv, comm, stream=None):
    hetccl_all_gather(_ptr(send), _ptr(recv), send.numel(), dtype_code(send.dtype), comm, _stream(stream, send))


def broadcast(send, recv, root, comm, stream=None):
    hetccl_broadcast(_ptr(send), _ptr(recv), recv.numel(), dtype_code(recv.dtype), root, comm, _stream(stream, recv))


def reduce(send, recv, root, comm, op="sum", stream=None):
    """recv may be None on non-root ranks."""
    hetccl_reduce(_ptr(send), _ptr(recv), send.numel(), dtype_code(send.dtype), op, root, comm, _stream(stream, send))


def all_to_all(send, recv, comm, stream=None):
    """send/recv hold nranks equal blocks."""
    n = hetccl_comm_info(comm)["nranks"]
    hetccl_all_to_all(_ptr(send), _ptr(recv), send.numel() // n, dtype_code(send.dtype), comm, _stream(stream, send))


def mux_reduce(sends, recvs, root, comm, op="sum", stream=None):
    hetccl_mux_reduce(sends, recvs, sends[0].numel(), dtype_code(sends[0].dtype), op, root, comm, _stream(stream, sends[0]))


def mux_all_to_all(sends, recvs, comm, stream=None):
    n = len(sends)
    hetccl_mux_all_to_all(sends, recvs, sends[0].numel() // n, dtype_code(sends[0].dtype), comm, _stream(stream, sends[0]))


def mux_allreduce(sends, recvs, comm, op="sum", stream=None):
    hetccl_mux_allreduce(sends, recvs, recvs[0].numel(), dtype_code(recvs[0].dtype), op, comm, _stream(stream, sends[0]))


def mux_reduce_scatter(sends, recvs, comm, op="sum", stream=None):
    hetccl_mux_reduce_scatter(sends, recvs, recvs[0].numel(), dtype_code(recvs[0].dtype), op, comm, _stream(stream, sends[0]))


def mux_all_gather(sends, recvs, comm, stream=None):
    hetccl_mux_all_gather(sends, recvs, sends[0].numel(), dtype_code(sends[0].dtype), comm, _stream(stream, sends[0]))


def mux_broadcast(sends, recvs, root, comm, stream=None):
    hetccl_mux_broadcast(sends, recvs, recvs[0].numel(), dtype_code(recvs[0].dtype), root, comm, _stream(stream, sends[0]))
