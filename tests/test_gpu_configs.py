"""BASELINE.json's configs at their full sizes, rank-multiplexed on one B200 (the driver's box), in the launch
configuration bench.py times (hetccl_comm_init_mux defaults): every output is compared with the CPU oracle on
sampled windows — the oracle computes each window from the same seeded inputs regenerated at that offset — or in
full where the oracle finishes in seconds. SURVEY §8(d): C1 fp32 1 Mi elements 1+1; C2 bf16 256 MiB per rank 4+4;
C3 bf16 RS 256 MiB + AG on 2+6; C4 1.3B-parameter gradients' 25 MiB buckets on 2+2+4 (first buckets and the
ragged tail); C5 Llama-7B's 256 MiB buckets and its ragged tail on 1+1 / 2+2 / 4+4."""
import numpy as np
import pytest

import oracle
import synth
from harness import MAPS, assert_matches, to_numpy

pytestmark = pytest.mark.gpu

W = 4096  # elements per sampled window


def _windows(count, k=12, seed=0):
    rng = np.random.default_rng(seed)
    starts = sorted({0, count - W, count // 2} | {int(v) for v in rng.integers(0, count - W, k)})
    return [s for s in starts if 0 <= s <= count - W]


def _bf16_dev(seed, rank, count):
    import torch
    x = synth.normal(seed, rank, count, "bf16")
    return torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to("cuda")


def _run_ar(m, count, seed, what):
    import torch
    import paper_2601_22585_b200 as hc
    n = len(m)
    comm = hc.hetccl_comm_init_mux(n, m, 0)
    try:
        sends = [_bf16_dev(seed, r, count) for r in range(n)]
        recvs = [torch.empty_like(s) for s in sends]
        hc.mux_allreduce(sends, recvs, comm)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        del sends
        for st in _windows(count, seed=seed):
            xs = [synth.normal(seed, r, W, "bf16", start=st) for r in range(n)]
            want = oracle.allreduce(xs, m, "bf16", "sum")
            for r in range(n):
                assert_matches(to_numpy(recvs[r][st:st + W], "bf16"), want, xs, "bf16", "sum", f"{what} @{st} rank {r}")
    finally:
        hc.hetccl_comm_destroy(comm)


def test_c1_fp32_1mi_mux_bitexact():
    """C1: fp32 sum of 1 Mi elements on 1+1, uniform and ramp inputs, the whole output bitwise."""
    import torch
    import paper_2601_22585_b200 as hc
    m = MAPS["1+1"]
    count = 1 << 20
    comm = hc.hetccl_comm_init_mux(2, m, 0)
    try:
        for xs in ([synth.uniform(1, r, count) for r in range(2)], [synth.ramp(r, count) for r in range(2)]):
            sends = [torch.from_numpy(x.copy()).cuda() for x in xs]
            recvs = [torch.empty_like(s) for s in sends]
            hc.mux_allreduce(sends, recvs, comm)
            torch.cuda.synchronize()
            want = oracle.allreduce(xs, m, "f32", "sum")
            for r in range(2):
                assert np.array_equal(to_numpy(recvs[r], "f32").view(np.uint32), want.view(np.uint32))
    finally:
        hc.hetccl_comm_destroy(comm)


def test_c2_4p4_256mib():
    """C2's target point, the bench's workload: 4+4, 256 MiB bf16 per rank (seed 2)."""
    _run_ar(MAPS["4+4"], 256 * (1 << 20) // 2, 2, "C2 4+4 256 MiB")


def test_c3_2p6_rs_ag_256mib():
    """C3: reduce-scatter of 256 MiB per rank on 2+6 (recvcount 16,777,216), then all-gather of the shards."""
    import torch
    import paper_2601_22585_b200 as hc
    m = MAPS["2+6"]
    n = len(m)
    count = 256 * (1 << 20) // 2
    R = count // n
    comm = hc.hetccl_comm_init_mux(n, m, 0)
    try:
        sends = [_bf16_dev(3, r, count) for r in range(n)]
        shards = [torch.empty(R, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
        hc.mux_reduce_scatter(sends, shards, comm)
        torch.cuda.synchronize()
        del sends
        outs = [torch.empty(count, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
        hc.mux_all_gather(shards, outs, comm)
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        for r in range(n):
            for st in _windows(R, k=3, seed=r):
                xs = [synth.normal(3, q, W, "bf16", start=r * R + st) for q in range(n)]
                want = oracle.allreduce(xs, m, "bf16", "sum")  # block r of the reduction
                assert_matches(to_numpy(shards[r][st:st + W], "bf16"), want, xs, "bf16", "sum", f"C3 RS rank {r} @{st}")
        sh = [to_numpy(s, "bf16") for s in shards]
        for r in (0, n - 1):
            got = to_numpy(outs[r], "bf16")
            assert np.array_equal(got, np.concatenate(sh)), f"C3 AG rank {r}"
    finally:
        hc.hetccl_comm_destroy(comm)


def test_c4_2p2p4_buckets():
    """C4: 25 MiB buckets (13,107,200 elements) of the 1.3e9-parameter gradients on 2+2+4, bucket 0 in full and the
    ragged tail bucket (2,387,200 elements) in full, both bitwise against the oracle."""
    import torch
    import paper_2601_22585_b200 as hc
    m = MAPS["2+2+4"]
    n = len(m)
    comm = hc.hetccl_comm_init_mux(n, m, 0)
    try:
        for count, seed in ((13_107_200, 4), (2_387_200, 40)):
            xs = [synth.normal(seed, r, count, "bf16") for r in range(n)]
            sends = [torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to("cuda") for x in xs]
            recvs = [torch.empty_like(s) for s in sends]
            hc.mux_allreduce(sends, recvs, comm)
            torch.cuda.synchronize()
            want = oracle.allreduce_threaded(xs, m, "bf16", "sum")
            for r in range(n):
                assert_matches(to_numpy(recvs[r], "bf16"), want, xs, "bf16", "sum", f"C4 bucket of {count} rank {r}")
    finally:
        hc.hetccl_comm_destroy(comm)


@pytest.mark.parametrize("name", ["1+1", "2+2", "4+4"])
def test_c5_llama7b_buckets(name):
    """C5: Llama-7B's 256 MiB buckets (134,217,728 elements) and its ragged tail (27,529,216) at the bench's splits
    for 2 / 4 / 8 ranks."""
    m = MAPS[name]
    _run_ar(m, 134_217_728, 5, f"C5 {name} 256 MiB bucket")
    _run_ar(m, 27_529_216, 50, f"C5 {name} tail")
