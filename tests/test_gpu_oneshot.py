"""GPU parity of the one-shot small-message All-Reduce (NEXT-3, k_allreduce_oneshot): every rank pushes
its chunk to every peer and reduces all n operands in the oracle's domain-major order, so results must
be bit-identical to the oracle (and to the hierarchical path). Rank-multiplexed and one rank per GPU."""
import numpy as np
import pytest

import oracle
from harness import MAPS, assert_matches, inputs, to_numpy, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _env(monkeypatch):
    monkeypatch.setenv("HETCCL_TIMEOUT_S", "10")
    monkeypatch.setenv("HETCCL_ONESHOT_KB", "1024")


def _hc():
    import paper_2601_22585_b200 as hc
    return hc


def _run(name, dt, op, count, seed=41, kind="normal", comm=None):
    import torch
    hc = _hc()
    m = MAPS[name]
    n = len(m)
    xs = inputs(kind, seed, n, count, dt)
    own = comm is None
    comm = comm or hc.hetccl_comm_init_mux(n, m, 0)
    try:
        sends = [to_torch(x, dt, "cuda") for x in xs]
        recvs = [torch.full_like(s, 3) for s in sends]
        hc.mux_allreduce(sends, recvs, comm, op=op)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        want = oracle.allreduce(xs, m, dt, op)
        for r in range(n):
            assert_matches(to_numpy(recvs[r], dt), want, xs, dt, op, f"oneshot {name} {dt} {op} rank {r}")
    finally:
        if own:
            hc.hetccl_comm_destroy(comm)


@pytest.mark.parametrize("name", ["1+1", "2+2", "1+3", "1+1+2", "4+4", "2+6", "2+2+4", "8", "interleaved", "1+2+3"])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_oneshot_splits(name, dt):
    _run(name, dt, "sum", 70001)


@pytest.mark.parametrize("dt", ["int32", "f16", "f32", "bf16"])
@pytest.mark.parametrize("op", ["sum", "max", "min"])
def test_oneshot_dtypes_ops(dt, op):
    _run("2+2+4", dt, op, 12345, kind="bits" if dt == "int32" else "normal")


@pytest.mark.parametrize("count", [1, 2, 7, 8, 9, 4097, 262144])
def test_oneshot_ragged(count):
    _run("2+6", "bf16", "sum", count)


def test_oneshot_and_pipeline_interleaved(monkeypatch):
    """Double-buffered one-shot ops (> 2 in a row) interleaved with pipeline ops on one comm."""
    hc = _hc()
    m = MAPS["2+2+4"]
    comm = hc.hetccl_comm_init_mux(len(m), m, 0)
    try:
        for it, count in enumerate([1000, 5000, 300000, 777, 1 << 20, 64, 3, 200001, 9999]):
            _run("2+2+4", "bf16", "sum", count, seed=100 + it, comm=comm)
    finally:
        hc.hetccl_comm_destroy(comm)


@pytest.mark.multigpu
@pytest.mark.parametrize("name", ["1+1", "2+2", "1+3", "1+1+2"])
def test_oneshot_multi(name):
    import torch
    hc = _hc()
    m = MAPS[name]
    n = len(m)
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    comms = hc.hetccl_comm_init_all(list(range(n)), m)
    try:
        for it, count in enumerate([5, 4096 + 3, 250000]):
            xs = inputs("normal", 50 + it, n, count, "bf16")
            sends = [to_torch(xs[r], "bf16", f"cuda:{r}") for r in range(n)]
            recvs = [torch.empty_like(s) for s in sends]
            ss = [torch.cuda.Stream(device=i) for i in range(n)]
            for r in range(n):
                torch.cuda.synchronize(r)
            for r in range(n):
                hc.allreduce(sends[r], recvs[r], comms[r], stream=ss[r])
            for r in range(n):
                torch.cuda.synchronize(r)
            want = oracle.allreduce(xs, m, "bf16", "sum")
            for r in range(n):
                hc.hetccl_comm_get_async_error(comms[r])
                assert np.array_equal(to_numpy(recvs[r], "bf16"), want), f"{name} count {count} rank {r}"
    finally:
        for c in comms:
            hc.hetccl_comm_destroy(c)


@pytest.mark.multigpu
@pytest.mark.parametrize("name", ["1+1", "2+2", "1+1+2"])
def test_oneshot_multi_back_to_back_mixed_sizes(name):
    """one-shot ops of different sizes use different channel counts; enqueued back to back
    on every GPU with no host sync, a fast rank's next op must never overwrite a region a slow peer is still
    reading. Each channel now owns a private region, so its own parity + ACK order every reuse. Every op has
    its own output buffers and all results are checked after the whole sequence."""
    import torch
    hc = _hc()
    m = MAPS[name]
    n = len(m)
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    comms = hc.hetccl_comm_init_all(list(range(n)), m)
    try:
        sizes = [2000, 6000, 8192, 3000, 16000, 24577, 4096, 100, 70000, 5000] * 4
        cases = []
        for i, count in enumerate(sizes):
            xs = inputs("normal", 700 + i, n, count, "bf16")
            sends = [to_torch(xs[r], "bf16", f"cuda:{r}") for r in range(n)]
            recvs = [torch.empty_like(s) for s in sends]
            cases.append((xs, sends, recvs))
        streams = [torch.cuda.Stream(device=r) for r in range(n)]
        for r in range(n):
            torch.cuda.synchronize(r)
        for r in range(n):  # rank r enqueues its whole sequence before rank r+1 starts: maximal skew
            for xs, sends, recvs in cases:
                hc.allreduce(sends[r], recvs[r], comms[r], stream=streams[r])
        for r in range(n):
            torch.cuda.synchronize(r)
        for c in comms:
            hc.hetccl_comm_get_async_error(c)
        for i, (xs, sends, recvs) in enumerate(cases):
            want = oracle.allreduce(xs, m, "bf16", "sum")
            for r in range(n):
                assert np.array_equal(to_numpy(recvs[r], "bf16"), want), f"op {i} (count {sizes[i]}) rank {r}"
    finally:
        for c in comms:
            hc.hetccl_comm_destroy(c)
