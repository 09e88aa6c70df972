"""NVLS mode (opt-in HETCCL_NVLS=1): All-Reduce whose intra-domain stages run in the
NVSwitch through per-domain multicast objects (multimem.ld_reduce / multimem.st), single process driving
2 or 4 B200s. The switch's summation order inside a domain is not reading R3's, so the bar is the R7 gate
against an fp64 reference (bf16/fp16, staged in fp32 through the switch), an fp32 recursive-summation bound
(fp32), every rank bitwise identical, and exact results on integer-valued data (any order sums those
exactly)."""
import numpy as np
import pytest

import oracle
from harness import MAPS, as_f64, inputs, to_numpy, to_torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

NVLS_MAPS = ["2", "2+2", "4"]


def _ngpu():
    import torch
    return torch.cuda.device_count()


def _sync(n):
    import torch
    for i in range(n):
        torch.cuda.synchronize(i)


@pytest.fixture
def nvls_env(monkeypatch):
    monkeypatch.setenv("HETCCL_NVLS", "1")
    monkeypatch.setenv("HETCCL_TIMEOUT_S", "10")
    monkeypatch.setenv("HETCCL_NVLS_MB", "2")  # small chunks: multi-chunk ops at test sizes


def _comms(m):
    import paper_2601_22585_b200 as hc
    comms = hc.hetccl_comm_init_all(list(range(len(m))), m)
    on, ptr, nb = hc.hetccl_comm_nvls(comms[0])
    if not on:
        why = hc.lib().hetccl_get_last_error(comms[0])
        for c in comms:
            hc.hetccl_comm_destroy(c)
        pytest.skip(f"NVLS unavailable: {why}")
    return comms


def _check(got_list, xs, dt, what, m):
    F = np.stack([as_f64(x, dt) for x in xs])
    R = F.sum(0)
    A = np.abs(F).sum(0)
    n = len(xs)
    for r, got in enumerate(got_list):
        bad = np.nonzero(got != got_list[0])[0]
        assert bad.size == 0, f"{what}: rank {r} differs from rank 0 at {bad.size} elements, first {bad[:8].tolist()}"
    g = as_f64(got_list[0], dt)
    if dt == "f32":
        u = 2.0 ** -24
        assert np.all(np.abs(g - R) <= 2 * n * u * A + 1e-30), f"{what}: fp32 bound"
    else:
        # R7's gate unchanged (north_star / SURVEY §8(c) c7): 16-bit inputs are staged in fp32 through the
        # switch (its fp32 adds are RNE, q33/q34), each partial narrowed once, so the error bound is the
        # oracle's: |Y - R| <= (2 * 2^-p + gamma_{n-1}) * sum|x| < 1e-2 * sum|x|
        bad = np.nonzero(np.abs(g - R) > 1e-2 * A + 1e-30)[0]
        assert bad.size == 0, f"{what}: elementwise gate fails at {bad.size} elements, first {bad[:8].tolist()}"
        nrm = np.linalg.norm(R)
        if nrm > 0:
            assert np.linalg.norm(g - R) / nrm <= 1e-2, f"{what}: normwise gate"


@pytest.mark.parametrize("name", NVLS_MAPS)
@pytest.mark.parametrize("dt", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("count", [1, 7, 5 * 8192 + 333, (3 << 20) // 2 + 5])
def test_nvls_allreduce(name, dt, count, nvls_env):
    import paper_2601_22585_b200 as hc
    m = MAPS[name]
    n = len(m)
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    comms = _comms(m)
    try:
        for it in range(2):
            xs = inputs("normal", 31 + it, n, count, dt)
            sends = [to_torch(xs[r], dt, f"cuda:{r}") for r in range(n)]
            recvs = [s.clone().fill_(0) for s in sends]
            _sync(n)
            for r in range(n):
                hc.allreduce(sends[r], recvs[r], comms[r])
            _sync(n)
            for c in comms:
                hc.hetccl_comm_get_async_error(c)
            _check([to_numpy(y, dt) for y in recvs], xs, dt, f"{name} {dt} n={count} it={it}", m)
    finally:
        for c in comms:
            hc.hetccl_comm_destroy(c)


@pytest.mark.parametrize("name", NVLS_MAPS)
def test_nvls_exact_on_integers_and_inplace(name, nvls_env):
    """Small integers sum exactly in any order: NVLS equals the oracle bitwise; in place too."""
    import torch
    import paper_2601_22585_b200 as hc
    m = MAPS[name]
    n = len(m)
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    count = 3 * 65536 + 11
    rng = np.random.default_rng(5)
    xs = [rng.integers(-8, 9, count).astype(np.float32) for _ in range(n)]
    xs = [np.frombuffer(torch.from_numpy(x).bfloat16().view(torch.int16).numpy().tobytes(), np.uint16) for x in xs]
    comms = _comms(m)
    try:
        bufs = [to_torch(xs[r], "bf16", f"cuda:{r}") for r in range(n)]
        _sync(n)
        for r in range(n):
            hc.allreduce(bufs[r], bufs[r], comms[r])
        _sync(n)
        want = oracle.allreduce(xs, m, "bf16", "sum")
        for r in range(n):
            assert np.array_equal(to_numpy(bufs[r], "bf16"), want), f"{name} rank {r}"
    finally:
        for c in comms:
            hc.hetccl_comm_destroy(c)


@pytest.mark.parametrize("name", ["2", "2+2"])
def test_nvls_zero_copy_buffer(name, nvls_env):
    """In place on the comm's multicast-bound buffer (f32): no copies in or out; repeated ops (slot reuse).
    A 16-bit All-Reduce on it is rejected: the buffer is the fp32 staging area of 16-bit ops."""
    import torch
    import paper_2601_22585_b200 as hc
    m = MAPS[name]
    n = len(m)
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    comms = _comms(m)
    try:
        count = 65536 * 3
        for it in range(3):
            xs = inputs("normal", 40 + it, n, count, "f32")
            bufs = [hc.nvls_buffer(comms[r], count, torch.float32, r) for r in range(n)]
            for r in range(n):
                bufs[r].copy_(to_torch(xs[r], "f32", f"cuda:{r}"))
            _sync(n)
            for r in range(n):
                hc.allreduce(bufs[r], bufs[r], comms[r])
            _sync(n)
            _check([to_numpy(b, "f32") for b in bufs], xs, "f32", f"{name} zero-copy it={it}", m)
        b16 = hc.nvls_buffer(comms[0], count, torch.bfloat16, 0)
        with pytest.raises(hc.HetcclError) as ei:
            hc.allreduce(b16, b16, comms[0])
        assert ei.value.code == 4
    finally:
        for c in comms:
            hc.hetccl_comm_destroy(c)


def test_nvls_ineligible_map_stays_p2p(monkeypatch):
    """Unequal domains (1+3) or singleton domains (1+1): NVLS is not set up, All-Reduce stays bit-exact P2P."""
    import paper_2601_22585_b200 as hc
    monkeypatch.setenv("HETCCL_NVLS", "1")
    for name in ("1+1", "1+3"):
        m = MAPS[name]
        n = len(m)
        if _ngpu() < n:
            continue
        comms = hc.hetccl_comm_init_all(list(range(n)), m)
        try:
            assert hc.hetccl_comm_nvls(comms[0])[0] is False
            count = 4099
            xs = inputs("normal", 3, n, count, "bf16")
            sends = [to_torch(xs[r], "bf16", f"cuda:{r}") for r in range(n)]
            recvs = [s.clone() for s in sends]
            _sync(n)
            for r in range(n):
                hc.allreduce(sends[r], recvs[r], comms[r])
            _sync(n)
            want = oracle.allreduce(xs, m, "bf16", "sum")
            for r in range(n):
                assert np.array_equal(to_numpy(recvs[r], "bf16"), want)
        finally:
            for c in comms:
                hc.hetccl_comm_destroy(c)


def _nvls_rank(rank, world, port, m, q):
    import os
    import sys
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), HETCCL_NVLS="1", HETCCL_NVLS_MB="2",
                      HETCCL_TIMEOUT_S="20")
    import torch
    import torch.distributed as dist
    import paper_2601_22585_b200 as hc
    from harness import inputs, to_numpy, to_torch
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = hc.init_process_group_comm(m)
        on, _, _ = hc.hetccl_comm_nvls(comm)
        why = (hc.lib().hetccl_get_last_error(comm) or b"").decode()
        res = []
        if on:
            for dt, count in (("bf16", 5 * 8192 + 333), ("bf16", (3 << 20) // 2 + 5), ("f32", 65536 * 3 + 7)):
                for it in range(2):
                    xs = inputs("normal", 70 + it, world, count, dt)
                    x = to_torch(xs[rank], dt, "cuda")
                    y = torch.zeros_like(x)
                    hc.allreduce(x, y, comm)
                    torch.cuda.synchronize()
                    hc.hetccl_comm_get_async_error(comm)
                    res.append((dt, count, it, to_numpy(y, dt)))
        hc.hetccl_comm_destroy(comm)
        q.put((rank, bool(on), why, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["2", "2+2"])
def test_nvls_one_rank_per_process(name):
    """NVLS across processes (one rank per GPU): the domain leader hands its multicast handle to the members as a
    file descriptor over a unix socket, every member adds its device and binds its memory, and the ranks agree
    before the comm switches to NVLS. Results: every rank bitwise identical, R7's gate (16-bit staged in fp32)."""
    import socket
    import torch
    import torch.multiprocessing as mp
    m = MAPS[name]
    n = len(m)
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_nvls_rank, args=(r, n, port, m, q)) for r in range(n)]
    for p in ps:
        p.start()
    out = dict((r, (on, why, res)) for r, on, why, res in (q.get(timeout=300) for _ in range(n)))
    for p in ps:
        p.join(timeout=60)
    ons = {out[r][0] for r in range(n)}
    assert len(ons) == 1, f"ranks disagree on NVLS: {out}"
    if not ons.pop():
        pytest.skip(f"NVLS unavailable across processes: {out[0][1]}")
    for j, (dt, count, it, _) in enumerate(out[0][2]):
        xs = inputs("normal", 70 + it, n, count, dt)
        _check([out[r][2][j][3] for r in range(n)], xs, dt, f"{name} {dt} n={count} it={it} (multi-process)", m)
