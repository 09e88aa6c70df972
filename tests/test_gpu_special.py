"""Special values through the GPU path (R9-R11): subnormal operands and results are kept (no
flush-to-zero on either side), infinities propagate bit-exactly, NaNs are compared by class (payload bits
are unpinned, R10); int32 sums wrap (R8). Rank-multiplexed 2+2+4 and 1+3 splits, pipeline and one-shot."""
import numpy as np
import pytest

import oracle
from harness import MAPS, to_numpy, to_torch

pytestmark = pytest.mark.gpu


def _special_inputs(dt, n, count, seed):
    rng = np.random.default_rng(seed)
    if dt == "int32":
        vals = np.array([2**31 - 1, -2**31, 1, -1, 0, 2**30], np.int64)
        return [rng.choice(vals, count).astype(np.int32) for _ in range(n)]
    if dt == "f32":
        tiny = np.float32(1.4e-45)
        pool = np.array([tiny, -tiny, 3 * tiny, np.float32(1.1754942e-38), np.inf, -np.inf, np.nan, 0.0, -0.0, 1.0,
                         np.float32(3.4e38)], np.float32)
        return [rng.choice(pool, count, p=[.15, .15, .15, .15, .02, .02, .02, .1, .1, .1, .04]) for _ in range(n)]
    if dt == "f16":
        pool = np.array([6e-8, -6e-8, 1.2e-7, 6.1e-5, np.inf, -np.inf, np.nan, 0.0, -0.0, 1.0, 65000.0], np.float16)
        return [rng.choice(pool, count, p=[.15, .15, .15, .15, .02, .02, .02, .1, .1, .1, .04]) for _ in range(n)]
    # bf16 raw bits: subnormals (exponent 0), inf, nan, zeros, normals, huge
    pool = np.array([0x0001, 0x8001, 0x0003, 0x007f, 0x7f80, 0xff80, 0x7fc0, 0x0000, 0x8000, 0x3f80, 0x7f7f], np.uint16)
    return [rng.choice(pool, count, p=[.15, .15, .15, .15, .02, .02, .02, .1, .1, .1, .04]) for _ in range(n)]


def _isnan(a, dt):
    if dt == "bf16":
        return ((a & 0x7f80) == 0x7f80) & ((a & 0x007f) != 0)
    if dt == "int32":
        return np.zeros(a.shape, bool)
    return np.isnan(a)


@pytest.mark.parametrize("oneshot", ["0", "1024"])
@pytest.mark.parametrize("name", ["2+2+4", "1+3"])
@pytest.mark.parametrize("dt", ["f32", "f16", "bf16", "int32"])
def test_special_values(name, dt, oneshot, monkeypatch):
    import torch
    import paper_2601_22585_b200 as hc
    monkeypatch.setenv("HETCCL_ONESHOT_KB", oneshot)
    monkeypatch.setenv("HETCCL_TILE_KB", "16")
    m = MAPS[name]
    n = len(m)
    count = 30011
    xs = _special_inputs(dt, n, count, 5)
    comm = hc.hetccl_comm_init_mux(n, m, 0)
    try:
        sends = [to_torch(x, dt, "cuda") for x in xs]
        recvs = [torch.empty_like(s) for s in sends]
        hc.mux_allreduce(sends, recvs, comm)
        torch.cuda.synchronize()
        want = oracle.allreduce(xs, m, dt, "sum")
        wn = _isnan(want, dt)
        for r in range(n):
            got = to_numpy(recvs[r], dt)
            gn = _isnan(got, dt)
            assert np.array_equal(gn, wn), f"{name} {dt} rank {r}: NaN class differs"
            gb = got.view(np.uint16 if got.itemsize == 2 else np.uint32)
            wb = want.view(np.uint16 if want.itemsize == 2 else np.uint32)
            assert np.array_equal(gb[~wn], wb[~wn]), f"{name} {dt} rank {r}: non-NaN values differ"
    finally:
        hc.hetccl_comm_destroy(comm)


def test_buffers_must_be_device_memory_of_the_comm():
    """a host buffer (or one on another device) is hetcclInvalidUsage, checked before launch."""
    import torch
    import paper_2601_22585_b200 as hc
    comm = hc.hetccl_comm_init_mux(2, [0, 1], 0)
    try:
        dev = [torch.zeros(4096, device="cuda") for _ in range(2)]
        host = [torch.zeros(4096).pin_memory() for _ in range(2)]
        plain = [torch.zeros(4096) for _ in range(2)]
        for bad_s, bad_r in ((host, dev), (dev, host), (plain, dev)):
            with pytest.raises(hc.HetcclError) as ei:
                hc.mux_allreduce(bad_s, bad_r, comm)
            assert ei.value.code == 5, ei.value
        if torch.cuda.device_count() > 1:
            other = [torch.zeros(4096, device="cuda:1") for _ in range(2)]
            with pytest.raises(hc.HetcclError) as ei:
                hc.mux_allreduce(other, dev, comm)
            assert ei.value.code == 5
        hc.mux_allreduce(dev, dev, comm)  # still usable
        torch.cuda.synchronize()
    finally:
        hc.hetccl_comm_destroy(comm)
