"""Build libhetccl.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

The library is the C ABI of include/hetccl.h; the Python binding (``__init__.py``) loads it with
ctypes. Compiled with -lineinfo (ncu source view) and WITHOUT --use_fast_math (IEEE arithmetic,
no flush-to-zero: DESIGN.md reading R9).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhetccl.so")
# kernels.cu is compiled twice: as is (TMA movers, 4 CTAs per SM) and through kernels_legacy.cu (cp.async
# movers, 2 CTAs per SM); the translation units compile in parallel, then link into one library
SOURCES = ["kernels.cu", "kernels_legacy.cu", "runtime.cu", "plan.cpp", "nvls.cu"]
HEADERS = ["hetccl_internal.h", os.path.join("..", "..", "include", "hetccl.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CFLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
          "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden", "-Xptxas", "-v"]
LDFLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "--shared", "-cudart", "static"]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(f) > t for f in files)


def build(force=False, verbose=False, variant=None, defines=()):
    """Build libhetccl.so (or, for A/B experiments, libhetccl_<variant>.so with extra -D defines)."""
    lib = LIB if not variant else os.path.join(HERE, f"libhetccl_{variant}.so")
    if not force and not variant and not stale():
        return LIB
    tmp = lib + f".tmp{os.getpid()}"
    objdir = os.path.join(HERE, "build", variant or "default")
    os.makedirs(objdir, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *CFLAGS, *[f"-D{d}" for d in defines], "-c", "-o", obj, os.path.join(CSRC, src)]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    log = []
    failed = False
    for src, obj, p in procs:
        out, err = p.communicate()
        log.append(f"=== {src}\n{out}{err}")
        if p.returncode != 0:
            failed = True
            sys.stderr.write(out + err)
    if failed:
        raise RuntimeError("nvcc failed building libhetccl.so")
    p = subprocess.run([NVCC, *LDFLAGS, "-o", tmp] + [obj for _, obj, _ in procs], capture_output=True, text=True)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError("nvcc failed linking libhetccl.so")
    with open(os.path.join(HERE, "ptxas_info.txt" if not variant else f"ptxas_info_{variant}.txt"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        sys.stderr.write("\n".join(log))
    os.replace(tmp, lib)
    return lib


NCCL_INC = os.path.join(os.path.dirname(os.path.dirname(os.__file__)), "site-packages", "nvidia", "nccl", "include")
SHIM = os.path.join(HERE, "libhetccl_nccl.so")


def nccl_include():
    try:
        import nvidia.nccl as nn
        return os.path.join(list(nn.__path__)[0], "include")
    except Exception:
        return NCCL_INC


def build_shim(force=False):
    """libhetccl_nccl.so: LD_PRELOAD interposition of NCCL's collectives onto libhetccl.so (NEXT-4)."""
    src = os.path.join(CSRC, "nccl_shim.cpp")
    if not force and os.path.exists(SHIM) and os.path.getmtime(SHIM) > max(os.path.getmtime(src), os.path.getmtime(LIB)):
        return SHIM
    tmp = SHIM + f".tmp{os.getpid()}"
    cmd = [NVCC, "-O2", "-std=c++17", "-x", "cu", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler",
           "-fPIC,-fvisibility=hidden", "--shared", "-cudart", "static", f"-I{nccl_include()}", src, "-o", tmp,
           f"-L{HERE}", "-lhetccl", "-Xlinker", "-rpath,$ORIGIN", "-ldl"]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError("nvcc failed building libhetccl_nccl.so")
    os.replace(tmp, SHIM)
    return SHIM


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    build_shim(force="--force" in sys.argv)
    print(LIB, SHIM)
