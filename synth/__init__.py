"""Seeded synthetic inputs (the one module both the CUDA path's tests/bench and the oracle consume).

Holds none of the method's arithmetic: every element is a pure function of (seed, rank, index)
(splitmix64 counter hash in ``synth_gen.c``). Recipes:

* ``normal``  — N(0,1) * scale; gradient-like. bf16 by truncating binary32 bits; f16 via numpy cast.
* ``uniform`` — U[lo, hi).
* ``ramp``    — x_r[i] = (i mod M) + M*r  (closed-form All-Reduce, SURVEY §8(c) pins).
* ``bits``    — uniformly random int32 (exercises wrap-around).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth_gen.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None


def build(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64, i, sz, f, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_size_t, ctypes.c_float, ctypes.c_void_p
        L.synth_normal_f32.argtypes = [u64, i, sz, sz, f, vp]
        L.synth_normal_bf16.argtypes = [u64, i, sz, sz, f, vp]
        L.synth_uniform_f32.argtypes = [u64, i, sz, sz, f, f, vp]
        L.synth_bits_u32.argtypes = [u64, i, sz, sz, vp]
        _lib = L
    return _lib


NP = {"int32": np.int32, "f32": np.float32, "f16": np.float16, "bf16": np.uint16}


def normal(seed, rank, n, dtype="bf16", scale=1.0 / 16, start=0, out=None):
    """N(0,1)*scale per (seed, rank, index); SURVEY §8(d) uses scale 2^-4 for the gradient buckets."""
    if dtype == "bf16":
        out = np.empty(n, np.uint16) if out is None else out
        lib().synth_normal_bf16(seed, rank, start, n, scale, out.ctypes.data)
        return out
    f = np.empty(n, np.float32)
    lib().synth_normal_f32(seed, rank, start, n, scale, f.ctypes.data)
    if dtype == "f32":
        return f
    if dtype == "f16":
        return f.astype(np.float16)
    if dtype == "int32":
        return np.round(f * 1000).astype(np.int32)
    raise ValueError(dtype)


def uniform(seed, rank, n, dtype="f32", lo=-1.0, hi=1.0, start=0):
    f = np.empty(n, np.float32)
    lib().synth_uniform_f32(seed, rank, start, n, lo, hi, f.ctypes.data)
    if dtype == "f32":
        return f
    if dtype == "f16":
        return f.astype(np.float16)
    if dtype == "bf16":
        return (f.view(np.uint32) >> 16).astype(np.uint16)
    if dtype == "int32":
        return np.floor(f * 1e6).astype(np.int32)
    raise ValueError(dtype)


def bits(seed, rank, n, start=0):
    u = np.empty(n, np.uint32)
    lib().synth_bits_u32(seed, rank, start, n, u.ctypes.data)
    return u.view(np.int32)


def ramp(rank, n, M=4096, dtype="f32"):
    """x_r[i] = (i mod M) + M*r."""
    v = (np.arange(n, dtype=np.int64) % M) + M * rank
    if dtype == "int32":
        return v.astype(np.int32)
    if dtype == "f32":
        return v.astype(np.float32)
    if dtype == "f16":
        return v.astype(np.float16)
    if dtype == "bf16":  # values used with bf16 are small integers (exact in bf16)
        return (v.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    raise ValueError(dtype)


def make(kind, seed, rank, n, dtype, **kw):
    if kind == "normal":
        return normal(seed, rank, n, dtype, **kw)
    if kind == "uniform":
        return uniform(seed, rank, n, dtype, **kw)
    if kind == "bits":
        assert dtype == "int32"
        return bits(seed, rank, n)
    if kind == "ramp":
        return ramp(rank, n, dtype=dtype, **kw)
    raise ValueError(kind)
