"""CPU oracle for the hierarchical collectives — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package. The product path (``paper_2601_22585_b200``) never does; the two share
no code. The arithmetic lives in ``hetccl_oracle.c`` (plain C, see its header for the passages of
PAPER.md / SPEC.md it follows); this module only marshals numpy arrays.

Element representation on the Python side: int32 -> np.int32, f32 -> np.float32, f16 -> np.float16,
bf16 -> np.uint16 holding the raw bf16 bits.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hetccl_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

INT32, F16, F32, BF16 = 2, 6, 7, 9
SUM, MAX, MIN = 0, 2, 3
NP_DTYPE = {INT32: np.int32, F16: np.float16, F32: np.float32, BF16: np.uint16}
DTYPE_NAMES = {"int32": INT32, "f16": F16, "f32": F32, "bf16": BF16}
OP_NAMES = {"sum": SUM, "max": MAX, "min": MIN}

CFLAGS = ["-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared"]


def build(force=False):
    """Compile liboracle.so with gcc (no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "hetccl_oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, sz, i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
        pp = ctypes.POINTER(ctypes.c_void_p)
        ip = ctypes.POINTER(ctypes.c_int)
        L.oracle_allreduce.argtypes = [i, ip, pp, vp, sz, i, i]
        L.oracle_reduce_scatter.argtypes = [i, ip, pp, pp, sz, i, i]
        L.oracle_all_gather.argtypes = [i, pp, pp, sz, i]
        L.oracle_broadcast.argtypes = [i, i, pp, pp, sz, i]
        L.oracle_reduce.argtypes = [i, ip, i, pp, vp, sz, i, i]
        L.oracle_all_to_all.argtypes = [i, pp, pp, sz, i]
        for f in ("oracle_allreduce", "oracle_reduce_scatter", "oracle_all_gather", "oracle_broadcast",
                  "oracle_reduce", "oracle_all_to_all"):
            getattr(L, f).restype = i
        L.oracle_f32_to_bf16.argtypes = [ctypes.c_float]
        L.oracle_f32_to_bf16.restype = ctypes.c_uint16
        L.oracle_f32_to_f16.argtypes = [ctypes.c_float]
        L.oracle_f32_to_f16.restype = ctypes.c_uint16
        L.oracle_bf16_to_f32.argtypes = [ctypes.c_uint16]
        L.oracle_bf16_to_f32.restype = ctypes.c_float
        L.oracle_f16_to_f32.argtypes = [ctypes.c_uint16]
        L.oracle_f16_to_f32.restype = ctypes.c_float
        _lib = L
    return _lib


def _dt(dtype):
    return DTYPE_NAMES[dtype] if isinstance(dtype, str) else dtype


def _op(op):
    return OP_NAMES[op] if isinstance(op, str) else op


def _ptrs(arrays):
    arr = (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])
    return arr


def _map(m):
    return (ctypes.c_int * len(m))(*[int(v) for v in m])


def _check(xs, dt, count=None):
    want = NP_DTYPE[dt]
    out = []
    for x in xs:
        x = np.ascontiguousarray(x)
        if x.dtype != want:
            raise TypeError(f"oracle expects {np.dtype(want)} arrays for dtype {dt}, got {x.dtype}")
        if count is not None and x.size != count:
            raise ValueError("length mismatch across ranks")
        out.append(x)
    return out


def allreduce(xs, rank_to_domain, dtype, op="sum"):
    """Y (one array) — every rank's All-Reduce output."""
    dt, o = _dt(dtype), _op(op)
    xs = _check(xs, dt, xs[0].size)
    y = np.empty(xs[0].size, NP_DTYPE[dt])
    rc = lib().oracle_allreduce(len(xs), _map(rank_to_domain), _ptrs(xs), y.ctypes.data, y.size, dt, o)
    if rc:
        raise ValueError("oracle_allreduce: invalid argument")
    return y


def allreduce_threaded(xs, rank_to_domain, dtype, op="sum", threads=None):
    """allreduce() with the ELEMENTS split into `threads` contiguous ranges, each reduced by one host thread
    calling the same C routine on its range (ctypes releases the GIL). The per-element fold order is
    unchanged ("an optional T-thread variant splits elements only"), so Y is bit-identical to
    allreduce(). Used for the T = host-cores oracle timing beside the GPU."""
    from concurrent.futures import ThreadPoolExecutor
    dt, o = _dt(dtype), _op(op)
    xs = _check(xs, dt, xs[0].size)
    count = xs[0].size
    y = np.empty(count, NP_DTYPE[dt])
    T = max(1, min(int(threads or os.cpu_count() or 1), count))
    es = y.itemsize
    bounds = [count * t // T for t in range(T + 1)]
    m = _map(rank_to_domain)
    L = lib()

    def run(t):
        lo, hi = bounds[t], bounds[t + 1]
        if hi <= lo:
            return 0
        ptrs = (ctypes.c_void_p * len(xs))(*[x.ctypes.data + lo * es for x in xs])
        return L.oracle_allreduce(len(xs), m, ptrs, y.ctypes.data + lo * es, hi - lo, dt, o)

    with ThreadPoolExecutor(max_workers=T) as ex:
        rcs = list(ex.map(run, range(T)))
    if any(rcs):
        raise ValueError("oracle_allreduce: invalid argument")
    return y


def reduce_scatter(xs, rank_to_domain, dtype, op="sum"):
    """[y_0 .. y_{n-1}]: rank r's block r of the reduction (x_r holds n*recvcount elements)."""
    dt, o = _dt(dtype), _op(op)
    n = len(xs)
    xs = _check(xs, dt, xs[0].size)
    if xs[0].size % n:
        raise ValueError("sendcount must be nranks*recvcount")
    rc_ = xs[0].size // n
    ys = [np.empty(rc_, NP_DTYPE[dt]) for _ in range(n)]
    rc = lib().oracle_reduce_scatter(n, _map(rank_to_domain), _ptrs(xs), _ptrs(ys), rc_, dt, o)
    if rc:
        raise ValueError("oracle_reduce_scatter: invalid argument")
    return ys


def all_gather(xs, dtype):
    dt = _dt(dtype)
    n = len(xs)
    xs = _check(xs, dt, xs[0].size)
    ys = [np.empty(n * xs[0].size, NP_DTYPE[dt]) for _ in range(n)]
    if lib().oracle_all_gather(n, _ptrs(xs), _ptrs(ys), xs[0].size, dt):
        raise ValueError("oracle_all_gather: invalid argument")
    return ys


def broadcast(xs, root, dtype):
    dt = _dt(dtype)
    n = len(xs)
    xs = _check(xs, dt, xs[0].size)
    ys = [np.empty(xs[0].size, NP_DTYPE[dt]) for _ in range(n)]
    if lib().oracle_broadcast(n, root, _ptrs(xs), _ptrs(ys), xs[0].size, dt):
        raise ValueError("oracle_broadcast: invalid argument")
    return ys


def reduce(xs, rank_to_domain, root, dtype, op="sum"):
    dt, o = _dt(dtype), _op(op)
    xs = _check(xs, dt, xs[0].size)
    y = np.empty(xs[0].size, NP_DTYPE[dt])
    if lib().oracle_reduce(len(xs), _map(rank_to_domain), root, _ptrs(xs), y.ctypes.data, y.size, dt, o):
        raise ValueError("oracle_reduce: invalid argument")
    return y


def all_to_all(xs, dtype):
    dt = _dt(dtype)
    n = len(xs)
    xs = _check(xs, dt, xs[0].size)
    if xs[0].size % n:
        raise ValueError("count must be nranks*blockcount")
    b = xs[0].size // n
    ys = [np.empty(n * b, NP_DTYPE[dt]) for _ in range(n)]
    if lib().oracle_all_to_all(n, _ptrs(xs), _ptrs(ys), b, dt):
        raise ValueError("oracle_all_to_all: invalid argument")
    return ys


def f32_to_bf16(f):
    return lib().oracle_f32_to_bf16(float(f))


def f32_to_f16(f):
    return lib().oracle_f32_to_f16(float(f))


def bf16_to_f32(h):
    return lib().oracle_bf16_to_f32(int(h))


def f16_to_f32(h):
    return lib().oracle_f16_to_f32(int(h))
