"""GPU parity, rank-multiplexed mode: every logical rank of an n-rank domain split runs
inside ONE cooperative kernel on one B200, through the C ABI (hetccl_mux_*), with the same device
code and flag protocol as the one-rank-per-GPU path. Compared element by element with the oracle."""
import os

import numpy as np
import pytest

import oracle
from harness import MAPS, assert_matches, inputs, to_numpy, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _env(monkeypatch):
    monkeypatch.setenv("HETCCL_TIMEOUT_S", "10")
    monkeypatch.setenv("HETCCL_ONESHOT_KB", "0")  # these tests cover the hierarchical pipeline (test_gpu_oneshot.py the rest)


def _hc():
    import paper_2601_22585_b200 as hc
    return hc


def _run_ar(name, dt, op, count, tile_kb=None, nch=None, kind="normal", seed=1, inplace=False, monkeypatch=None):
    import torch
    hc = _hc()
    if tile_kb:
        monkeypatch.setenv("HETCCL_TILE_KB", str(tile_kb))
    if nch:
        monkeypatch.setenv("HETCCL_NCHANNELS", str(nch))
    m = MAPS[name]
    n = len(m)
    xs = inputs(kind, seed, n, count, dt)
    comm = hc.hetccl_comm_init_mux(n, m, 0)
    try:
        sends = [to_torch(x, dt, "cuda") for x in xs]
        recvs = sends if inplace else [torch.full_like(s, 7) for s in sends]
        hc.mux_allreduce(sends, recvs, comm, op=op)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        want = oracle.allreduce(xs, m, dt, op)
        for r in range(n):
            assert_matches(to_numpy(recvs[r], dt), want, xs, dt, op, f"{name} {dt} {op} rank {r}")
    finally:
        hc.hetccl_comm_destroy(comm)


@pytest.mark.parametrize("name", ["1+1", "2+2", "1+3", "1+1+2", "4+4", "2+6", "2+2+4", "8", "singletons4",
                                  "interleaved", "3+5", "1+2+3"])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_allreduce_splits(name, dt, monkeypatch):
    # 4 KiB tiles -> many tiles per channel, ragged last tile (count not a multiple of anything)
    _run_ar(name, dt, "sum", 3 * 4096 + 1000 + 3, tile_kb=4, monkeypatch=monkeypatch)


@pytest.mark.parametrize("dt", ["int32", "f16", "f32", "bf16"])
@pytest.mark.parametrize("op", ["sum", "max", "min"])
def test_allreduce_dtypes_ops(dt, op, monkeypatch):
    _run_ar("2+2+4", dt, op, 20000 + 13, tile_kb=8, kind="bits" if dt == "int32" else "normal", seed=3,
            monkeypatch=monkeypatch)


@pytest.mark.parametrize("count", [1, 2, 7, 8, 9, 63, 1000, 65536 + 5])
def test_allreduce_small_and_ragged(count, monkeypatch):
    _run_ar("2+6", "bf16", "sum", count, monkeypatch=monkeypatch)
    _run_ar("1+1", "f32", "sum", count, monkeypatch=monkeypatch)


def test_allreduce_inplace(monkeypatch):
    _run_ar("4+4", "bf16", "sum", 100003, tile_kb=16, inplace=True, monkeypatch=monkeypatch)


def test_allreduce_c1_config(monkeypatch):
    """BASELINE config 0: fp32 sum of 1 Mi elements over 2 ranks as 1+1 (ramp and uniform data)."""
    _run_ar("1+1", "f32", "sum", 1 << 20, kind="uniform", seed=1, monkeypatch=monkeypatch)
    _run_ar("1+1", "f32", "sum", 1 << 20, kind="ramp", monkeypatch=monkeypatch)


def test_repeated_calls_and_channel_changes(monkeypatch):
    """Counters are cumulative across launches: vary count/tile/channels between calls on one comm."""
    import torch
    hc = _hc()
    m = MAPS["2+2+4"]
    n = len(m)
    comm = hc.hetccl_comm_init_mux(n, m, 0)
    try:
        for it, (count, tkb) in enumerate([(5000, 4), (100000, 16), (17, 4), (300000, 64), (5000, 4)] * 3):
            monkeypatch.setenv("HETCCL_TILE_KB", str(tkb))
            xs = inputs("normal", 100 + it, n, count, "bf16")
            sends = [to_torch(x, "bf16", "cuda") for x in xs]
            recvs = [torch.empty_like(s) for s in sends]
            hc.mux_allreduce(sends, recvs, comm)
            torch.cuda.synchronize()
            want = oracle.allreduce(xs, m, "bf16", "sum")
            for r in range(n):
                assert_matches(to_numpy(recvs[r], "bf16"), want, xs, "bf16", "sum", f"iter {it} rank {r}")
        hc.hetccl_comm_get_async_error(comm)
    finally:
        hc.hetccl_comm_destroy(comm)


def test_n1_copy():
    import torch
    hc = _hc()
    comm = hc.hetccl_comm_init_mux(1, [0], 0)
    try:
        x = torch.randn(12345, device="cuda")
        y = torch.empty_like(x)
        hc.mux_allreduce([x], [y], comm)
        torch.cuda.synchronize()
        assert torch.equal(x, y)
    finally:
        hc.hetccl_comm_destroy(comm)


def test_trace_stamps_monotone(monkeypatch):
    """HETCCL_TRACE_ITERS: per-iteration stamps are ordered wait <= work <= end <= fenced."""
    import torch
    monkeypatch.setenv("HETCCL_TRACE_ITERS", "16")
    hc = _hc()
    m = MAPS["2+2"]
    comm = hc.hetccl_comm_init_mux(4, m, 0)
    try:
        xs = [torch.randn(1 << 20, device="cuda") for _ in range(4)]
        ys = [torch.empty_like(x) for x in xs]
        hc.mux_allreduce(xs, ys, comm)
        tr = hc.hetccl_comm_get_trace(comm)
        assert tr is not None and tr.shape[0] == 4 and tr.shape[3] == 10
        used = tr[..., 0] > 0
        assert used.any()
        for k in range(3):
            assert np.all(tr[..., k + 1][used] >= tr[..., k][used])
        # kernel entry <= first poll, last fence <= kernel exit (iteration 0 row, words 8 and 9)
        ch = used[..., 0]
        assert np.all(tr[..., 0, 8][ch] <= tr[..., 0, 0][ch]) and np.all(tr[..., 0, 9][ch] >= tr[..., 0, 3][ch])
    finally:
        hc.hetccl_comm_destroy(comm)


def test_cuda_graph_replay(monkeypatch):
    """The protocol keeps its cumulative targets on the device, so a captured All-Reduce (pipeline and
    one-shot) replays correctly many times; inputs change between replays."""
    import torch
    monkeypatch.setenv("HETCCL_ONESHOT_KB", "1024")
    hc = _hc()
    m = MAPS["2+2+4"]
    n = len(m)
    comm = hc.hetccl_comm_init_mux(n, m, 0)
    try:
        for count in (100003, 3 * (1 << 20) + 5):  # one-shot (default cutoff), then pipeline
            xs0 = inputs("normal", 200, n, count, "bf16")
            sends = [to_torch(x, "bf16", "cuda") for x in xs0]
            recvs = [torch.empty_like(s) for s in sends]
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                hc.mux_allreduce(sends, recvs, comm, stream=s)  # warm-up outside the graph
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                hc.mux_allreduce(sends, recvs, comm, stream=s)
            for it in range(12):
                xs = inputs("normal", 300 + it, n, count, "bf16")
                for r in range(n):
                    sends[r].copy_(to_torch(xs[r], "bf16", "cuda"))
                g.replay()
                torch.cuda.synchronize()
                want = oracle.allreduce(xs, m, "bf16", "sum")
                for r in range(n):
                    assert np.array_equal(to_numpy(recvs[r], "bf16"), want), f"replay {it} count {count} rank {r}"
        hc.hetccl_comm_get_async_error(comm)
    finally:
        hc.hetccl_comm_destroy(comm)


@pytest.mark.parametrize("direct,final_wait,pull,flat", [("0", "1", "0", "0"), ("1", "0", "0", "0"), ("1", "1", "0", "0"),
                                                        ("1", "1", "1", "0"), ("1", "1", "0", "1"), ("1", "1", "1", "1")])
@pytest.mark.parametrize("name", ["2+2", "1+3", "4+4", "2+6", "2+2+4", "8", "1+1"])
def test_allreduce_direct_and_staged(name, direct, final_wait, pull, flat, monkeypatch):
    """Rank-multiplexed comms write final pieces straight into every rank's recv buffer (HETCCL_DIRECT=1,
    default) — in place too; HETCCL_DIRECT=0 keeps the staged path of the multi-GPU mode."""
    monkeypatch.setenv("HETCCL_DIRECT", direct)
    monkeypatch.setenv("HETCCL_FINAL_WAIT", final_wait)
    monkeypatch.setenv("HETCCL_PULL", pull)
    monkeypatch.setenv("HETCCL_FLAT_AG", flat)
    _run_ar(name, "bf16", "sum", 70001, tile_kb=16, monkeypatch=monkeypatch)
    _run_ar(name, "f32", "sum", 50021, tile_kb=16, inplace=True, monkeypatch=monkeypatch)
