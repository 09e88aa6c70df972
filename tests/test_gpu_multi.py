"""GPU parity, one rank per GPU (single process driving 2 or 4 B200s over NVLink peer access via
hetccl_comm_init_all): each rank's kernel runs on its own GPU and pushes into peers' scratch over
NVSwitch. Compared element by element with the oracle."""
import numpy as np
import pytest

import oracle
from harness import MAPS, assert_matches, inputs, to_numpy, to_torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


@pytest.fixture(autouse=True)
def _env(monkeypatch):
    monkeypatch.setenv("HETCCL_TIMEOUT_S", "10")
    monkeypatch.setenv("HETCCL_ONESHOT_KB", "0")  # these tests cover the hierarchical pipeline (test_gpu_oneshot.py the rest)


def _ngpu():
    import torch
    return torch.cuda.device_count()


def _comms(m):
    import paper_2601_22585_b200 as hc
    return hc.hetccl_comm_init_all(list(range(len(m))), m)


def _streams(n):
    import torch
    return [torch.cuda.Stream(device=i) for i in range(n)]


def _sync(n):
    import torch
    for i in range(n):
        torch.cuda.synchronize(i)


MULTI_MAPS = ["1+1", "2", "2+2", "1+3", "1+1+2", "4", "singletons4"]


@pytest.mark.parametrize("name", MULTI_MAPS)
@pytest.mark.parametrize("dt,op", [("bf16", "sum"), ("f32", "sum"), ("int32", "sum"), ("f16", "max")])
def test_allreduce_multi(name, dt, op, monkeypatch):
    import paper_2601_22585_b200 as hc
    m = MAPS[name]
    n = len(m)
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    monkeypatch.setenv("HETCCL_TILE_KB", "16")
    count = 5 * 8192 + 333
    xs = inputs("bits" if dt == "int32" else "normal", 11, n, count, dt)
    comms = _comms(m)
    try:
        ss = _streams(n)
        sends = [to_torch(xs[r], dt, f"cuda:{r}") for r in range(n)]
        recvs = [s.clone().fill_(0) for s in sends]
        _sync(n)
        for r in range(n):
            hc.allreduce(sends[r], recvs[r], comms[r], op=op, stream=ss[r])
        _sync(n)
        for r in range(n):
            hc.hetccl_comm_get_async_error(comms[r])
        want = oracle.allreduce(xs, m, dt, op)
        for r in range(n):
            assert_matches(to_numpy(recvs[r], dt), want, xs, dt, op, f"{name} rank {r}")
    finally:
        for c in comms:
            hc.hetccl_comm_destroy(c)


def test_c1_fp32_1mi_bitexact():
    """BASELINE config 0 on two real GPUs: fp32 sum, 1 Mi elements, 1+1 — bit-exact vs the oracle."""
    import paper_2601_22585_b200 as hc
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    m = MAPS["1+1"]
    for kind in ("uniform", "ramp"):
        xs = inputs(kind, 1, 2, 1 << 20, "f32")
        comms = _comms(m)
        try:
            sends = [to_torch(xs[r], "f32", f"cuda:{r}") for r in range(2)]
            recvs = [s.clone() for s in sends]
            for r in range(2):
                with __import__("torch").cuda.device(r):
                    hc.allreduce(sends[r], recvs[r], comms[r])
            _sync(2)
            want = oracle.allreduce(xs, m, "f32", "sum")
            for r in range(2):
                np.testing.assert_array_equal(to_numpy(recvs[r], "f32").view(np.uint32), want.view(np.uint32))
        finally:
            for c in comms:
                hc.hetccl_comm_destroy(c)


@pytest.mark.parametrize("name", ["1+1", "2+2", "1+3", "1+1+2", "4"])
@pytest.mark.parametrize("inplace,pull,flat", [(False, "-1", "0"), (True, "-1", "0"), (True, "1", "0"), (False, "-1", "1")])
def test_allreduce_symmetric_direct(name, inplace, pull, flat, monkeypatch):
    """Symmetric recv buffers (hetccl_mem_*): final pieces are written straight into the peers' buffers;
    results bitwise equal to the oracle, at an offset inside the buffer, in and out of place."""
    import torch
    import paper_2601_22585_b200 as hc
    m = MAPS[name]
    n = len(m)
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    monkeypatch.setenv("HETCCL_TILE_KB", "16")
    monkeypatch.setenv("HETCCL_ONESHOT_KB", "0")
    monkeypatch.setenv("HETCCL_PULL", pull)  # in place: the send buffer is symmetric too, so 1 = pull mode
    monkeypatch.setenv("HETCCL_FLAT_AG", flat)
    count, off = 5 * 8192 + 333, 1000
    xs = inputs("normal", 17, n, count, "bf16")
    comms = _comms(m)
    try:
        bufs = hc.symmetric_empty_all(comms, count + 2 * off, torch.bfloat16)
        for it in range(3):
            xs = inputs("normal", 17 + it, n, count, "bf16")
            sends = []
            for r in range(n):
                bufs[r].fill_(0)
                if inplace:
                    bufs[r][off:off + count].copy_(to_torch(xs[r], "bf16", f"cuda:{r}"))
                    sends.append(bufs[r][off:off + count])
                else:
                    sends.append(to_torch(xs[r], "bf16", f"cuda:{r}"))
            _sync(n)
            for r in range(n):
                with torch.cuda.device(r):
                    hc.allreduce(sends[r], bufs[r][off:off + count], comms[r])
            _sync(n)
            want = oracle.allreduce(xs, m, "bf16", "sum")
            for r in range(n):
                hc.hetccl_comm_get_async_error(comms[r])
                assert np.array_equal(to_numpy(bufs[r][off:off + count], "bf16"), want), f"{name} it {it} rank {r}"
                assert not to_numpy(bufs[r][:off], "bf16").any(), "wrote outside the recv range"
    finally:
        for c in comms:
            hc.hetccl_comm_destroy(c)


def test_two_comms_two_streams_concurrently(monkeypatch):
    """C4's pattern: independent All-Reduces on two streams, one communicator per stream, channel counts
    that fit the SMs together (148 + 148 of 296 co-resident CTAs); results bitwise equal to the oracle."""
    import torch
    import paper_2601_22585_b200 as hc
    m = MAPS["2+2"] if _ngpu() >= 4 else MAPS["1+1"]
    n = len(m)
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    monkeypatch.setenv("HETCCL_NCHANNELS", "148")
    monkeypatch.setenv("HETCCL_ONESHOT_KB", "0")
    monkeypatch.setenv("HETCCL_TILE_KB", "64")
    ca = hc.hetccl_comm_init_all(list(range(n)), m)
    cb = hc.hetccl_comm_init_all(list(range(n)), m)
    try:
        count = 3 * (1 << 20) + 11
        xa = inputs("normal", 61, n, count, "bf16")
        xb = inputs("normal", 62, n, count, "bf16")
        sa = [torch.cuda.Stream(device=r) for r in range(n)]
        sb = [torch.cuda.Stream(device=r) for r in range(n)]
        ta = [to_torch(xa[r], "bf16", f"cuda:{r}") for r in range(n)]
        tb = [to_torch(xb[r], "bf16", f"cuda:{r}") for r in range(n)]
        ya = [torch.empty_like(t) for t in ta]
        yb = [torch.empty_like(t) for t in tb]
        _sync(n)
        for it in range(4):
            for r in range(n):
                hc.allreduce(ta[r], ya[r], ca[r], stream=sa[r])
                hc.allreduce(tb[r], yb[r], cb[r], stream=sb[r])
        _sync(n)
        wa = oracle.allreduce(xa, m, "bf16", "sum")
        wb = oracle.allreduce(xb, m, "bf16", "sum")
        for r in range(n):
            hc.hetccl_comm_get_async_error(ca[r])
            hc.hetccl_comm_get_async_error(cb[r])
            assert np.array_equal(to_numpy(ya[r], "bf16"), wa), f"stream a rank {r}"
            assert np.array_equal(to_numpy(yb[r], "bf16"), wb), f"stream b rank {r}"
    finally:
        for c in ca + cb:
            hc.hetccl_comm_destroy(c)


@pytest.mark.parametrize("name", ["1+1", "2+2", "1+3", "1+1+2", "4"])
@pytest.mark.parametrize("kernels", ["tma_s2g", "tma_st"])
def test_collectives_on_tma_kernels(name, kernels, monkeypatch):
    """One rank per GPU on the TMA kernel build (HETCCL_LEGACY=0; the default there is the legacy build): ring
    movers with bulk-copy stores to NVLink peers (S2G) and with per-thread stores. All-Reduce (staged and
    direct into symmetric buffers), Reduce-Scatter and All-Gather bitwise against the oracle."""
    import torch
    import paper_2601_22585_b200 as hc
    m = MAPS[name]
    n = len(m)
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    monkeypatch.setenv("HETCCL_LEGACY", "0")
    monkeypatch.setenv("HETCCL_S2G", "1" if kernels == "tma_s2g" else "0")
    monkeypatch.setenv("HETCCL_NCHANNELS", "64")
    count = (1 << 20) + 4099
    xs = inputs("normal", 81, n, count, "bf16")
    comms = _comms(m)
    try:
        ss = _streams(n)
        sends = [to_torch(xs[r], "bf16", f"cuda:{r}") for r in range(n)]
        recvs = [torch.zeros_like(s) for s in sends]
        sym_x = hc.symmetric_empty_all(comms, count, torch.bfloat16)
        sym_y = hc.symmetric_empty_all(comms, count, torch.bfloat16)
        for r in range(n):
            sym_x[r].copy_(sends[r])
        _sync(n)
        for r in range(n):
            hc.allreduce(sends[r], recvs[r], comms[r], stream=ss[r])
        for r in range(n):
            hc.allreduce(sym_x[r], sym_y[r], comms[r], stream=ss[r])
        _sync(n)
        want = oracle.allreduce(xs, m, "bf16", "sum")
        for r in range(n):
            assert_matches(to_numpy(recvs[r], "bf16"), want, xs, "bf16", "sum", f"{kernels} {name} staged rank {r}")
            assert_matches(to_numpy(sym_y[r], "bf16"), want, xs, "bf16", "sum", f"{kernels} {name} direct rank {r}")
        R = count // n
        rs = [torch.zeros(R, dtype=torch.bfloat16, device=f"cuda:{r}") for r in range(n)]
        for r in range(n):
            hc.reduce_scatter(sends[r][: n * R], rs[r], comms[r], stream=ss[r])
        _sync(n)
        blk = oracle.reduce_scatter([x[: n * R] for x in xs], m, "bf16", "sum")
        ag = [torch.zeros(n * R, dtype=torch.bfloat16, device=f"cuda:{r}") for r in range(n)]
        for r in range(n):
            assert np.array_equal(to_numpy(rs[r], "bf16"), blk[r]), f"{kernels} {name} RS rank {r}"
            hc.all_gather(rs[r], ag[r], comms[r], stream=ss[r])
        _sync(n)
        for r in range(n):
            assert np.array_equal(to_numpy(ag[r], "bf16"), np.concatenate(blk)), f"{kernels} {name} AG rank {r}"
        for c in comms:
            hc.hetccl_comm_get_async_error(c)
    finally:
        for c in comms:
            hc.hetccl_comm_destroy(c)
