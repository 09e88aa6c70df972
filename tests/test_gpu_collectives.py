"""GPU parity of the hierarchical Reduce-Scatter, All-Gather (a7) and Broadcast (a8)
through the C ABI, rank-multiplexed on one B200 (hetccl_mux_*) and one rank per GPU
(hetccl_comm_init_all), compared element by element with the oracle; plus AR == AG∘RS bitwise on the
GPU path (SURVEY §8(c) "Always" row)."""
import numpy as np
import pytest

import oracle
from harness import MAPS, assert_matches, inputs, to_numpy, to_torch

pytestmark = pytest.mark.gpu

SPLITS = ["1+1", "2+2", "1+3", "1+1+2", "4+4", "2+6", "2+2+4", "8", "interleaved", "1+2+3", "3+5"]


@pytest.fixture(autouse=True)
def _env(monkeypatch):
    monkeypatch.setenv("HETCCL_TIMEOUT_S", "10")
    monkeypatch.setenv("HETCCL_ONESHOT_KB", "0")  # these tests cover the hierarchical pipeline (test_gpu_oneshot.py the rest)


def _hc():
    import paper_2601_22585_b200 as hc
    return hc


def _mux(m):
    return _hc().hetccl_comm_init_mux(len(m), m, 0)


# ------------------------------------------------------------------------------ reduce-scatter
def _run_rs(name, dt, op, recvcount, kind="normal", seed=5, inplace=False):
    import torch
    hc = _hc()
    m = MAPS[name]
    n = len(m)
    xs = inputs(kind, seed, n, n * recvcount, dt)
    comm = _mux(m)
    try:
        sends = [to_torch(x, dt, "cuda") for x in xs]
        if inplace:
            recvs = [s[r * recvcount:(r + 1) * recvcount] for r, s in enumerate(sends)]
        else:
            recvs = [torch.full((recvcount,), 3, dtype=sends[0].dtype, device="cuda") for _ in range(n)]
        hc.mux_reduce_scatter(sends, recvs, comm, op=op)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        want = oracle.reduce_scatter(xs, m, dt, op)
        for r in range(n):
            blk = [x[r * recvcount:(r + 1) * recvcount] for x in xs]
            assert_matches(to_numpy(recvs[r], dt), want[r], blk, dt, op, f"RS {name} {dt} {op} rank {r}")
    finally:
        hc.hetccl_comm_destroy(comm)


@pytest.mark.parametrize("name", SPLITS)
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_reduce_scatter_splits(name, dt, monkeypatch):
    monkeypatch.setenv("HETCCL_TILE_KB", "8")
    _run_rs(name, dt, "sum", 3 * 1024 + 517)


@pytest.mark.parametrize("dt", ["int32", "f16", "f32", "bf16"])
@pytest.mark.parametrize("op", ["sum", "max", "min"])
def test_reduce_scatter_dtypes_ops(dt, op, monkeypatch):
    monkeypatch.setenv("HETCCL_TILE_KB", "16")
    _run_rs("2+6", dt, op, 4099, kind="bits" if dt == "int32" else "normal")


@pytest.mark.parametrize("recvcount", [1, 7, 8, 9, 1000, 70001])
def test_reduce_scatter_ragged(recvcount):
    _run_rs("2+2+4", "bf16", "sum", recvcount)


def test_reduce_scatter_inplace(monkeypatch):
    monkeypatch.setenv("HETCCL_TILE_KB", "16")
    _run_rs("2+6", "bf16", "sum", 20011, inplace=True)


# ------------------------------------------------------------------------------ all-gather
def _run_ag(name, dt, sendcount, inplace=False, seed=6):
    import torch
    hc = _hc()
    m = MAPS[name]
    n = len(m)
    xs = inputs("normal" if dt != "int32" else "bits", seed, n, sendcount, dt)
    comm = _mux(m)
    try:
        if inplace:
            recvs = [torch.zeros(n * sendcount, dtype=to_torch(xs[0][:1], dt, "cpu").dtype, device="cuda")
                     for _ in range(n)]
            sends = []
            for r in range(n):
                v = recvs[r][r * sendcount:(r + 1) * sendcount]
                v.copy_(to_torch(xs[r], dt, "cuda"))
                sends.append(v)
        else:
            sends = [to_torch(x, dt, "cuda") for x in xs]
            recvs = [torch.full((n * sendcount,), 5, dtype=sends[0].dtype, device="cuda") for _ in range(n)]
        hc.mux_all_gather(sends, recvs, comm)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        want = oracle.all_gather(xs, dt)
        for r in range(n):
            got = to_numpy(recvs[r], dt)
            assert np.array_equal(got.view(np.uint8), want[r].view(np.uint8)), f"AG {name} {dt} rank {r}"
    finally:
        hc.hetccl_comm_destroy(comm)


@pytest.mark.parametrize("name", SPLITS)
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_all_gather_splits(name, dt, monkeypatch):
    monkeypatch.setenv("HETCCL_TILE_KB", "8")
    _run_ag(name, dt, 3 * 1024 + 517)


@pytest.mark.parametrize("sendcount", [1, 7, 8, 9, 1000, 70001])
@pytest.mark.parametrize("dt", ["int32", "f16"])
def test_all_gather_ragged(sendcount, dt):
    _run_ag("2+2+4", dt, sendcount)


def test_all_gather_inplace(monkeypatch):
    monkeypatch.setenv("HETCCL_TILE_KB", "16")
    _run_ag("2+6", "bf16", 20011, inplace=True)


# ------------------------------------------------------------------------------ broadcast
def _run_bc(name, dt, count, root, inplace=False, seed=8):
    import torch
    hc = _hc()
    m = MAPS[name]
    n = len(m)
    xs = inputs("normal" if dt != "int32" else "bits", seed, n, count, dt)
    comm = _mux(m)
    try:
        sends = [to_torch(x, dt, "cuda") for x in xs]
        recvs = sends if inplace else [torch.full_like(s, 9) for s in sends]
        hc.mux_broadcast(sends, recvs, root, comm)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        want = oracle.broadcast(xs, root, dt)
        for r in range(n):
            got = to_numpy(recvs[r], dt)
            assert np.array_equal(got.view(np.uint8), want[r].view(np.uint8)), f"BC {name} root {root} rank {r}"
    finally:
        hc.hetccl_comm_destroy(comm)


@pytest.mark.parametrize("name", SPLITS)
@pytest.mark.parametrize("root_sel", ["first", "last", "mid"])
def test_broadcast_splits(name, root_sel, monkeypatch):
    monkeypatch.setenv("HETCCL_TILE_KB", "8")
    n = len(MAPS[name])
    root = {"first": 0, "last": n - 1, "mid": n // 2}[root_sel]
    _run_bc(name, "bf16", 5 * 1024 + 333, root)


@pytest.mark.parametrize("count", [1, 7, 9, 1000, 100003])
def test_broadcast_ragged(count):
    _run_bc("2+2+4", "f32", count, 5)


def test_broadcast_inplace(monkeypatch):
    monkeypatch.setenv("HETCCL_TILE_KB", "16")
    _run_bc("4+4", "int32", 50001, 6, inplace=True)


# ------------------------------------------------------------------------------ AR == AG o RS
@pytest.mark.parametrize("name", ["2+6", "2+2+4", "1+2+3"])
def test_ar_equals_ag_of_rs(name, monkeypatch):
    import torch
    hc = _hc()
    monkeypatch.setenv("HETCCL_TILE_KB", "16")
    m = MAPS[name]
    n = len(m)
    R = 4096 + 77
    xs = inputs("normal", 21, n, n * R, "bf16")
    comm = _mux(m)
    try:
        sends = [to_torch(x, "bf16", "cuda") for x in xs]
        ar = [torch.empty_like(s) for s in sends]
        hc.mux_allreduce(sends, ar, comm)
        rs = [torch.empty(R, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
        hc.mux_reduce_scatter(sends, rs, comm)
        ag = [torch.empty(n * R, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
        hc.mux_all_gather(rs, ag, comm)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        for r in range(n):
            assert torch.equal(ar[r].view(torch.int16), ag[r].view(torch.int16)), f"{name} rank {r}"
    finally:
        hc.hetccl_comm_destroy(comm)


# ------------------------------------------------------------------------------ one rank per GPU
def _ngpu():
    import torch
    return torch.cuda.device_count()


MULTI = ["1+1", "2+2", "1+3", "1+1+2", "4", "singletons4"]


@pytest.mark.multigpu
@pytest.mark.parametrize("name", MULTI)
@pytest.mark.parametrize("coll", ["rs", "ag", "bc"])
def test_collectives_multi(name, coll, monkeypatch):
    import torch
    hc = _hc()
    m = MAPS[name]
    n = len(m)
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    monkeypatch.setenv("HETCCL_TILE_KB", "16")
    comms = hc.hetccl_comm_init_all(list(range(n)), m)
    try:
        ss = [torch.cuda.Stream(device=i) for i in range(n)]
        if coll == "rs":
            R = 3 * 4096 + 71
            xs = inputs("normal", 31, n, n * R, "bf16")
            sends = [to_torch(xs[r], "bf16", f"cuda:{r}") for r in range(n)]
            recvs = [torch.empty(R, dtype=torch.bfloat16, device=f"cuda:{r}") for r in range(n)]
            for r in range(n):
                torch.cuda.synchronize(r)
            for r in range(n):
                hc.reduce_scatter(sends[r], recvs[r], comms[r], stream=ss[r])
            want = oracle.reduce_scatter(xs, m, "bf16", "sum")
        elif coll == "ag":
            C = 3 * 4096 + 71
            xs = inputs("normal", 32, n, C, "bf16")
            sends = [to_torch(xs[r], "bf16", f"cuda:{r}") for r in range(n)]
            recvs = [torch.empty(n * C, dtype=torch.bfloat16, device=f"cuda:{r}") for r in range(n)]
            for r in range(n):
                torch.cuda.synchronize(r)
            for r in range(n):
                hc.all_gather(sends[r], recvs[r], comms[r], stream=ss[r])
            want = oracle.all_gather(xs, "bf16")
        else:
            C = 5 * 4096 + 71
            root = n - 1
            xs = inputs("normal", 33, n, C, "bf16")
            sends = [to_torch(xs[r], "bf16", f"cuda:{r}") for r in range(n)]
            recvs = [torch.empty_like(s) for s in sends]
            for r in range(n):
                torch.cuda.synchronize(r)
            for r in range(n):
                hc.broadcast(sends[r], recvs[r], root, comms[r], stream=ss[r])
            want = oracle.broadcast(xs, root, "bf16")
        for r in range(n):
            torch.cuda.synchronize(r)
        for r in range(n):
            hc.hetccl_comm_get_async_error(comms[r])
            got = to_numpy(recvs[r], "bf16")
            assert np.array_equal(got, want[r]), f"{coll} {name} rank {r}"
    finally:
        for c in comms:
            hc.hetccl_comm_destroy(c)


# ------------------------------------------------------------------------------ reduce / all-to-all (NEXT-2)
def _run_reduce(name, dt, op, count, root, kind="normal", seed=61, inplace=False):
    import torch
    hc = _hc()
    m = MAPS[name]
    n = len(m)
    xs = inputs(kind, seed, n, count, dt)
    comm = _mux(m)
    try:
        sends = [to_torch(x, dt, "cuda") for x in xs]
        recvs = [s if inplace else torch.full_like(s, 7) for s in sends]
        hc.mux_reduce(sends, recvs, root, comm, op=op)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        want = oracle.reduce(xs, m, root, dt, op)
        assert_matches(to_numpy(recvs[root], dt), want, xs, dt, op, f"reduce {name} {dt} {op} root {root}")
        # the oracle's Reduce is the All-Reduce result (same order)
        assert np.array_equal(want.view(np.uint8), oracle.allreduce(xs, m, dt, op).view(np.uint8))
    finally:
        hc.hetccl_comm_destroy(comm)


@pytest.mark.parametrize("name", SPLITS)
@pytest.mark.parametrize("root_sel", ["first", "last", "mid"])
def test_reduce_splits(name, root_sel, monkeypatch):
    monkeypatch.setenv("HETCCL_TILE_KB", "8")
    n = len(MAPS[name])
    root = {"first": 0, "last": n - 1, "mid": n // 2}[root_sel]
    _run_reduce(name, "bf16", "sum", 5 * 1024 + 333, root)


@pytest.mark.parametrize("dt", ["int32", "f16", "f32", "bf16"])
@pytest.mark.parametrize("op", ["sum", "max", "min"])
def test_reduce_dtypes_ops(dt, op, monkeypatch):
    monkeypatch.setenv("HETCCL_TILE_KB", "16")
    _run_reduce("2+2+4", dt, op, 20011, 3, kind="bits" if dt == "int32" else "normal")


@pytest.mark.parametrize("count", [1, 7, 9, 1000, 100003])
def test_reduce_ragged_and_inplace(count):
    _run_reduce("2+6", "f32", "sum", count, 7)
    _run_reduce("4+4", "bf16", "sum", count, 2, inplace=True)


def _run_a2a(name, dt, block, seed=71):
    import torch
    hc = _hc()
    m = MAPS[name]
    n = len(m)
    xs = inputs("normal" if dt != "int32" else "bits", seed, n, n * block, dt)
    comm = _mux(m)
    try:
        sends = [to_torch(x, dt, "cuda") for x in xs]
        recvs = [torch.full_like(s, 4) for s in sends]
        hc.mux_all_to_all(sends, recvs, comm)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        want = oracle.all_to_all(xs, dt)
        for r in range(n):
            assert np.array_equal(to_numpy(recvs[r], dt).view(np.uint8), want[r].view(np.uint8)), f"a2a {name} rank {r}"
    finally:
        hc.hetccl_comm_destroy(comm)


@pytest.mark.parametrize("name", ["1+1", "2+2", "1+3", "4+4", "2+6", "2+2+4", "8", "interleaved"])
@pytest.mark.parametrize("dt", ["f32", "bf16", "int32"])
def test_all_to_all(name, dt, monkeypatch):
    monkeypatch.setenv("HETCCL_TILE_KB", "8")
    _run_a2a(name, dt, 3 * 1024 + 517)


@pytest.mark.parametrize("block", [1, 7, 8, 9, 70001])
def test_all_to_all_ragged(block):
    _run_a2a("2+2+4", "f16", block)


@pytest.mark.multigpu
@pytest.mark.parametrize("name", ["1+1", "2+2", "1+3"])
def test_reduce_a2a_multi(name, monkeypatch):
    import torch
    hc = _hc()
    m = MAPS[name]
    n = len(m)
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    monkeypatch.setenv("HETCCL_TILE_KB", "16")
    comms = hc.hetccl_comm_init_all(list(range(n)), m)
    try:
        C = 5 * 4096 + 71
        root = n - 1
        xs = inputs("normal", 81, n, n * C, "bf16")
        sends = [to_torch(xs[r], "bf16", f"cuda:{r}") for r in range(n)]
        red = [torch.empty_like(s) if r == root else None for r, s in enumerate(sends)]
        a2a = [torch.empty_like(s) for s in sends]
        for r in range(n):
            torch.cuda.synchronize(r)
        for r in range(n):
            with torch.cuda.device(r):
                hc.reduce(sends[r], red[r], root, comms[r])
                hc.all_to_all(sends[r], a2a[r], comms[r])
        for r in range(n):
            torch.cuda.synchronize(r)
        want_r = oracle.reduce(xs, m, root, "bf16", "sum")
        want_a = oracle.all_to_all(xs, "bf16")
        assert np.array_equal(to_numpy(red[root], "bf16"), want_r)
        for r in range(n):
            hc.hetccl_comm_get_async_error(comms[r])
            assert np.array_equal(to_numpy(a2a[r], "bf16"), want_a[r]), f"a2a {name} rank {r}"
    finally:
        for c in comms:
            hc.hetccl_comm_destroy(c)
