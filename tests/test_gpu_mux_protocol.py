"""The one-rank-per-GPU protocol variants, run rank-multiplexed on ONE B200 (VERDICT r1 "next" #1).

A driver box has one GPU, so the multi-GPU tests skip there. These tests run the SAME device code the
multi-GPU path runs, with the knobs it uses, inside one cooperative launch over all logical ranks:
  * HETCCL_SYS_SCOPE=1: the .sys-scope flag protocol (fence.acq_rel.sys, red.relaxed.sys, ld.acquire.sys)
    that ranks on different GPUs use, instead of the .gpu scope of rank-multiplexed comms;
  * HETCCL_PULL=0: push mode (peers store into my scratch; the multi-GPU default);
  * HETCCL_DIRECT=0: staged delivery through scratch (one rank per GPU with plain torch buffers);
    DIRECT=1 + FLAT_AG=0: the symmetric-buffer path at large sizes (direct recv, forwarding stage D);
  * HETCCL_TILE_KB=256: the multi-GPU default tile (rank-multiplexed comms default to 1 MiB);
  * HETCCL_WS=0 / 2: plain and warp-specialised pipelines.
Few channels (HETCCL_NCHANNELS=8) make every channel walk several tiles and the slot ring wrap. Every
result is compared element by element (bitwise) with the oracle.

What cannot be emulated on one GPU: the IPC bootstrap (hetccl_comm_export/connect needs two processes,
and two processes whose kernels wait on each other on ONE GPU are not guaranteed to be co-scheduled —
B200_PROFILING.md reports Xid 109 for exactly that), and NVLink-remote loads/stores (every address here
is local HBM). Those run in tests/test_gpu_multi.py on >= 2 GPUs and in the gloo tests on CPU.
"""
import numpy as np
import pytest

import oracle
from harness import MAPS, assert_matches, inputs, to_numpy, to_torch

pytestmark = pytest.mark.gpu

PROTOS = {
    "sys_push_staged": {"HETCCL_SYS_SCOPE": "1", "HETCCL_PULL": "0", "HETCCL_DIRECT": "0"},
    "sys_push_direct": {"HETCCL_SYS_SCOPE": "1", "HETCCL_PULL": "0", "HETCCL_DIRECT": "1", "HETCCL_FLAT_AG": "0"},
    "sys_push_flat": {"HETCCL_SYS_SCOPE": "1", "HETCCL_PULL": "0", "HETCCL_DIRECT": "1", "HETCCL_FLAT_AG": "1"},
    "sys_pull_direct": {"HETCCL_SYS_SCOPE": "1", "HETCCL_PULL": "1", "HETCCL_DIRECT": "1"},
    # warp-specialised: consumers sit 2 positions after producers, so the ring must exceed 2*(stages-1)+2
    "sys_push_staged_ws2": {"HETCCL_SYS_SCOPE": "1", "HETCCL_PULL": "0", "HETCCL_DIRECT": "0", "HETCCL_WS": "2",
                            "HETCCL_NSLOTS": "12"},
    "gpu_pull_ws2": {"HETCCL_SYS_SCOPE": "0", "HETCCL_WS": "2", "HETCCL_NSLOTS": "12"},
    # C-stage chunk stealing (opt-in): one tile per channel so jobs are published and taken by other channels
    "gpu_pull_steal": {"HETCCL_SYS_SCOPE": "0", "HETCCL_STEAL": "100", "HETCCL_TILE_KB": "4096"},
    "sys_push_direct_steal": {"HETCCL_SYS_SCOPE": "1", "HETCCL_PULL": "0", "HETCCL_DIRECT": "1", "HETCCL_STEAL": "25",
                              "HETCCL_TILE_KB": "4096"},
}
SPLITS = ["1+1", "2+2", "4+4", "2+6", "2+2+4", "1+2+3"]


@pytest.fixture(autouse=True)
def _env(monkeypatch):
    monkeypatch.setenv("HETCCL_TIMEOUT_S", "10")
    monkeypatch.setenv("HETCCL_ONESHOT_KB", "0")
    monkeypatch.setenv("HETCCL_TILE_KB", "256")
    monkeypatch.setenv("HETCCL_NCHANNELS", "8")


def _setup(proto, monkeypatch):
    for k, v in PROTOS[proto].items():
        monkeypatch.setenv(k, v)
    import paper_2601_22585_b200 as hc
    return hc


# 256 KiB tiles x 8 channels = 2 MiB per round: ~2.3 rounds per rank plus a ragged tail
COUNT_BF16 = 2 * (1 << 20) + 300_007
COUNT_F32 = (1 << 20) + 150_011


@pytest.mark.parametrize("proto", list(PROTOS))
@pytest.mark.parametrize("name", SPLITS)
def test_allreduce_protocols(proto, name, monkeypatch):
    import torch
    hc = _setup(proto, monkeypatch)
    m = MAPS[name]
    n = len(m)
    comm = hc.hetccl_comm_init_mux(n, m, 0)
    try:
        for dt, op, count, kind in (("bf16", "sum", COUNT_BF16, "normal"), ("f32", "sum", COUNT_F32, "uniform"),
                                    ("int32", "max", COUNT_F32, "bits")):
            xs = inputs(kind, 11, n, count, dt)
            sends = [to_torch(x, dt, "cuda") for x in xs]
            recvs = [torch.full_like(s, 7) for s in sends]
            hc.mux_allreduce(sends, recvs, comm, op=op)
            torch.cuda.synchronize()
            hc.hetccl_comm_get_async_error(comm)
            want = oracle.allreduce(xs, m, dt, op)
            for r in range(n):
                assert_matches(to_numpy(recvs[r], dt), want, xs, dt, op, f"{proto} {name} {dt} {op} rank {r}")
    finally:
        hc.hetccl_comm_destroy(comm)


@pytest.mark.parametrize("proto", ["sys_push_staged", "sys_push_staged_ws2"])
@pytest.mark.parametrize("name", ["2+2", "2+6", "2+2+4"])
def test_rs_ag_bcast_protocols(proto, name, monkeypatch):
    """RS / AG / Broadcast never take the direct or pull paths; .sys scope and WS are what differs."""
    import torch
    hc = _setup(proto, monkeypatch)
    m = MAPS[name]
    n = len(m)
    comm = hc.hetccl_comm_init_mux(n, m, 0)
    try:
        R = (1 << 18) + 4099  # per-shard elements: several 256 KiB shard tiles per channel
        xs = inputs("normal", 12, n, n * R, "bf16")
        sends = [to_torch(x, "bf16", "cuda") for x in xs]
        recvs = [torch.full((R,), 3, dtype=sends[0].dtype, device="cuda") for _ in range(n)]
        hc.mux_reduce_scatter(sends, recvs, comm)
        torch.cuda.synchronize()
        want = oracle.reduce_scatter(xs, m, "bf16", "sum")
        for r in range(n):
            blk = [x[r * R:(r + 1) * R] for x in xs]
            assert_matches(to_numpy(recvs[r], "bf16"), want[r], blk, "bf16", "sum", f"RS {proto} {name} rank {r}")
        # all-gather of the shards
        outs = [torch.full((n * R,), 5, dtype=sends[0].dtype, device="cuda") for _ in range(n)]
        hc.mux_all_gather(recvs, outs, comm)
        torch.cuda.synchronize()
        ag_want = oracle.all_gather([to_numpy(r_, "bf16") for r_ in recvs], "bf16")
        for r in range(n):
            assert np.array_equal(to_numpy(outs[r], "bf16"), ag_want[r]), f"AG {proto} {name} rank {r}"
        # broadcast from the last rank
        root = n - 1
        count = COUNT_BF16
        xb = inputs("normal", 13, n, count, "bf16")
        bs = [to_torch(x, "bf16", "cuda") for x in xb]
        br = [torch.full_like(b, 9) for b in bs]
        hc.mux_broadcast(bs, br, root, comm)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        for r in range(n):
            assert np.array_equal(to_numpy(br[r], "bf16"), xb[root]), f"BC {proto} {name} rank {r}"
    finally:
        hc.hetccl_comm_destroy(comm)


@pytest.mark.parametrize("proto", ["sys_push_staged", "sys_pull_direct", "gpu_pull_ws2"])
def test_back_to_back_no_host_sync(proto, monkeypatch):
    """Mixed sizes and ops enqueued back to back on one stream with no host synchronisation in between:
    the slot ring, the cumulative per-channel counters and the one-shot regions must carry over between
    launches whose channel counts differ. Every output buffer is distinct so all results are checked."""
    import torch
    monkeypatch.setenv("HETCCL_ONESHOT_KB", "512")  # small ops take the one-shot kernel, larger the pipeline
    hc = _setup(proto, monkeypatch)
    m = MAPS["2+2+4"]
    n = len(m)
    comm = hc.hetccl_comm_init_mux(n, m, 0)
    try:
        sizes = [4000, 6001, 8192, 100_003, 3000, 250_000, 600_001, 12_000, 9, 300_000] * 2
        cases = []
        for i, count in enumerate(sizes):
            xs = inputs("normal", 500 + i, n, count, "bf16")
            sends = [to_torch(x, "bf16", "cuda") for x in xs]
            recvs = [torch.empty_like(s) for s in sends]
            cases.append((xs, sends, recvs))
        torch.cuda.synchronize()
        for xs, sends, recvs in cases:
            hc.mux_allreduce(sends, recvs, comm)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        for i, (xs, sends, recvs) in enumerate(cases):
            want = oracle.allreduce(xs, m, "bf16", "sum")
            for r in range(n):
                got = to_numpy(recvs[r], "bf16")
                assert np.array_equal(got, want), f"op {i} (count {sizes[i]}) rank {r}"
    finally:
        hc.hetccl_comm_destroy(comm)
