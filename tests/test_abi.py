"""CPU-side checks of the C ABI (tests -m "not gpu"): the library loads without a GPU, exports every
symbol include/hetccl.h declares, validates maps, and its plan's per-rank byte counts equal the
closed forms of SURVEY §8(d) (no compute calls)."""
import ctypes
import os
import re
from fractions import Fraction

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hc():
    from paper_2601_22585_b200 import build
    build.build()
    import paper_2601_22585_b200 as hc
    return hc


def _declared():
    src = open(os.path.join(ROOT, "include", "hetccl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hetccl_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(hc):
    lib = hc.lib()
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(hc.EXPORTED)


def test_version_and_error_strings(hc):
    v = ctypes.c_int()
    assert hc.lib().hetccl_get_version(ctypes.byref(v)) == 0 and v.value == 100
    for code in range(6):
        assert hc.lib().hetccl_get_error_string(code)


@pytest.mark.parametrize("m,D", [([0, 1], 2), ([0, 0, 1, 1, 2, 2, 2, 2], 3), ([1, 0], 2), ([0] * 16, 1)])
def test_validate_map_ok(hc, m, D):
    assert hc.hetccl_validate_map(m) == D


@pytest.mark.parametrize("m", [[1, 1], [0, 2], [-1, 0], [0] * 17, []])
def test_validate_map_rejects(hc, m):
    with pytest.raises(hc.HetcclError):
        if not m:
            hc._check(hc.lib().hetccl_validate_map(0, None, None))
        else:
            hc.hetccl_validate_map(m)


def test_null_and_bad_args_without_gpu(hc):
    lib = hc.lib()
    assert lib.hetccl_allreduce(None, None, 4, 9, 0, None, None) == 4  # null comm
    info = hc.PlanInfo()
    assert lib.hetccl_plan_info(2, hc._imap([0, 1]), 0, 9, 16, 9, 0, 0, ctypes.byref(info)) == 4  # bad op
    assert lib.hetccl_plan_info(2, hc._imap([0, 1]), 0, 0, 16, 5, 0, 0, ctypes.byref(info)) == 4  # bad dtype
    assert lib.hetccl_plan_info(2, hc._imap([0, 1]), 0, 3, 16, 9, 2, 0, ctypes.byref(info)) == 4  # bad root
    assert lib.hetccl_plan_info(2, hc._imap([0, 1]), 0, 4, 16, 9, 5, 0, ctypes.byref(info)) == 4  # reduce: bad root
    # every entry point rejects a null communicator with hetcclInvalidArgument (no CUDA needed)
    p = ctypes.c_void_p()
    assert lib.hetccl_reduce(None, None, 4, 9, 0, 0, None, None) == 4
    assert lib.hetccl_all_to_all(None, None, 4, 9, None, None) == 4
    assert lib.hetccl_reduce_scatter(None, None, 4, 9, 0, None, None) == 4
    assert lib.hetccl_all_gather(None, None, 4, 9, None, None) == 4
    assert lib.hetccl_broadcast(None, None, 4, 9, 0, None, None) == 4
    assert lib.hetccl_mem_alloc(None, 1024, ctypes.byref(p)) == 4
    assert lib.hetccl_mem_free(None, None) == 4
    assert lib.hetccl_mem_connect(None, None, None, 0) == 4
    assert lib.hetccl_comm_destroy(None) == 4
    assert lib.hetccl_comm_get_async_error(None) == 4
    assert lib.hetccl_comm_nvls(None, None, None, None) == 4
    shape = (ctypes.c_int * 3)()
    assert lib.hetccl_comm_get_trace(None, None, 0, shape) == 4
    assert lib.hetccl_get_last_error(None) == b"null comm"


SPLITS = {"1+1": [0, 1], "2+2": [0, 0, 1, 1], "1+3": [0, 1, 1, 1], "1+1+2": [0, 1, 2, 2],
          "4+4": [0] * 4 + [1] * 4, "2+6": [0, 0] + [1] * 6, "2+2+4": [0, 0, 1, 1, 2, 2, 2, 2], "8": [0] * 8}


@pytest.fixture
def unbalanced(monkeypatch):
    """Whole-tile closed forms: keep the target tile (HETCCL_BALANCE=0) so count = k * tile stays whole."""
    monkeypatch.setenv("HETCCL_BALANCE", "0")


@pytest.mark.parametrize("name", sorted(SPLITS))
def test_allreduce_bytes_closed_form(hc, name, unbalanced):
    """Per-rank AR bytes = S*(2(d-1)/d + 2(D-1)/(D d)) for a count divisible by everything."""
    m = SPLITS[name]
    n, D = len(m), max(m) + 1
    # a whole number of full tiles (the ragged last tile is split on the clipped full-tile grid)
    tile = hc.hetccl_plan_info(m, 0, hc.OP_ALLREDUCE, 1 << 30, hc.BFLOAT16)["tile_elems"]
    count = tile * 1000
    S = count * 2
    busiest = 0
    for r in range(n):
        d = m.count(m[r])
        want = S * (Fraction(2 * (d - 1), d) + Fraction(2 * (D - 1), D * d))
        info = hc.hetccl_plan_info(m, r, hc.OP_ALLREDUCE, count, hc.BFLOAT16)
        assert info["bytes_sent"] == want and info["bytes_recv"] == want, (r, info, want)
        busiest = max(busiest, want)
    flat = Fraction(2 * (n - 1), n) * S
    table = {"1+1": 1, "2+2": 1, "1+3": Fraction(9, 10), "1+1+2": Fraction(9, 10), "4+4": 1,
             "2+6": Fraction(21, 22), "2+2+4": Fraction(21, 22), "8": 1}
    assert flat / busiest == table[name]


@pytest.mark.parametrize("name", ["2+6", "4+4", "1+3", "2+2+4"])
def test_rs_ag_bytes_closed_form(hc, name, unbalanced):
    """RS received per rank = (d-1)/d*S + (D-1)*S/n; AG is the mirror (sent = that); SURVEY §8(d)."""
    m = SPLITS[name]
    n, D = len(m), max(m) + 1
    tile = hc.hetccl_plan_info(m, 0, hc.OP_REDUCE_SCATTER, 1 << 28, hc.BFLOAT16)["tile_elems"]
    R = tile * 1000  # recvcount: whole tiles
    S = n * R * 2
    for r in range(n):
        d = m.count(m[r])
        recv = S * (Fraction(d - 1, d) + Fraction(D - 1, n))
        sent = S * Fraction(n - 1, n)
        rs = hc.hetccl_plan_info(m, r, hc.OP_REDUCE_SCATTER, R, hc.BFLOAT16)
        ag = hc.hetccl_plan_info(m, r, hc.OP_ALL_GATHER, R, hc.BFLOAT16)
        assert rs["bytes_recv"] == recv and rs["bytes_sent"] == sent, (r, rs)
        assert ag["bytes_sent"] == recv and ag["bytes_recv"] == sent, (r, ag)


def test_rs_2p6_survey_numbers(hc, unbalanced):
    """C3 (2+6): 2-domain ranks receive 0.625 S, 6-domain ranks 0.958 S."""
    m = SPLITS["2+6"]
    R = 16777216
    S = 8 * R * 2
    r0 = hc.hetccl_plan_info(m, 0, hc.OP_REDUCE_SCATTER, R, hc.BFLOAT16)["bytes_recv"]
    r7 = hc.hetccl_plan_info(m, 7, hc.OP_REDUCE_SCATTER, R, hc.BFLOAT16)["bytes_recv"]
    assert abs(r0 / S - 5 / 8) < 1e-4  # 16-byte rounding of the 1/6 pieces moves a few bytes
    assert abs(r7 / S - 23 / 24) < 1e-4


def test_conservation(hc):
    """Bytes sent over all ranks == bytes received over all ranks, any op, ragged counts."""
    for name, m in SPLITS.items():
        for op in range(6):
            for count in (1, 999, 123457):
                s = sum(hc.hetccl_plan_info(m, r, op, count, hc.BFLOAT16, root=len(m) - 1)["bytes_sent"]
                        for r in range(len(m)))
                v = sum(hc.hetccl_plan_info(m, r, op, count, hc.BFLOAT16, root=len(m) - 1)["bytes_recv"]
                        for r in range(len(m)))
                assert s == v, (name, op, count)


def test_single_domain_has_no_cross_traffic_and_singletons_no_intra(hc, unbalanced):
    """SPEC.md:400 analog: one domain -> only intra bytes (flat 2(n-1)/n S); all-singleton domains ->
    only the cross exchange (2(D-1)/D S)."""
    for m in ([0] * 4, [0, 1, 2, 3]):
        count = hc.hetccl_plan_info(m, 0, hc.OP_ALLREDUCE, 1 << 28, hc.FLOAT32)["tile_elems"] * 1000  # whole tiles
        S = count * 4
        assert hc.hetccl_plan_info(m, 0, hc.OP_ALLREDUCE, count, hc.FLOAT32)["bytes_sent"] == S * 3 // 2


# ------------------------------------------------------------------ pipeline schedule (host plan)
SCHED_MAPS = [[0, 1], [0, 0], [0, 0, 1, 1], [0, 1, 1, 1], [0, 1, 2, 2], [0, 0, 0, 0], [0, 1, 2, 3],
              [0, 0, 0, 0, 1, 1, 1, 1], [0, 0, 1, 1, 1, 1, 1, 1], [0, 0, 1, 1, 2, 2, 2, 2], [1, 0, 1, 0, 2, 2],
              [0, 0, 0, 1, 1, 1, 1, 1], [0, 1, 1, 2, 2, 2], [0] * 8, list(range(8)), [0, 1] * 8]


@pytest.mark.parametrize("m", SCHED_MAPS, ids=lambda m: "".join(map(str, m)))
@pytest.mark.parametrize("op", [0, 1, 2, 3, 4, 5])
def test_schedule_is_symmetric_and_acyclic(hc, m, op):
    """The flag protocol's invariants (kernels.cu run_pipeline): every signal a rank sends is awaited
    by its receiver on the same counter, every wait has a sender, a producer stage always precedes
    its consumer (so no iteration waits on itself), each counter has one consumer stage, active
    stages agree on every rank, and `writes` covers every rank signalled."""
    n = len(m)
    roots = range(n) if op in (3, 4) else [0]
    for root in roots:
        plans = [hc.hetccl_plan_stages(m, r, op, root) for r in range(n)]
        assert len({p["active"] for p in plans}) == 1
        act = plans[0]["active"]
        for w, pw in enumerate(plans):
            consumers = {}
            for s in range(pw["nstages"]):
                if pw["wait_ctr"][s] != 7:
                    assert (act >> s) & 1
                    assert pw["wait_ctr"][s] not in consumers, "two stages wait on one counter"
                    consumers[pw["wait_ctr"][s]] = s
            for s in range(pw["nstages"]):
                c, mask = pw["sig_ctr"][s], pw["sig_mask"][s]
                if c == 7:
                    assert mask == 0
                    continue
                assert (act >> s) & 1
                assert not (mask >> w) & 1, "no self signal"
                assert (pw["writes"] & mask) == mask
                for r in range(n):
                    if not (mask >> r) & 1:
                        continue
                    pr = plans[r]
                    cons = [s2 for s2 in range(pr["nstages"]) if pr["wait_ctr"][s2] == c]
                    assert len(cons) == 1, f"rank {r} never waits on counter {c}"
                    assert (pr["wait_mask"][cons[0]] >> w) & 1, f"rank {r} does not expect {w} on {c}"
                    assert cons[0] > s, "consumer must follow producer"
            for s in range(pw["nstages"]):
                c, mask = pw["wait_ctr"][s], pw["wait_mask"][s]
                for r in range(n):
                    if (mask >> r) & 1:
                        ps = plans[r]
                        assert any(ps["sig_ctr"][s2] == c and (ps["sig_mask"][s2] >> w) & 1
                                   for s2 in range(ps["nstages"])), f"{w} waits on {r} that never signals {c}"


def test_schedule_stage_sets(hc):
    # 1+1: no intra stages; one domain: no cross stage; singletons of 4: no intra stages
    assert hc.hetccl_plan_stages([0, 1], 0, 0)["active"] == 0b01110
    assert hc.hetccl_plan_stages([0, 0, 0, 0], 0, 0)["active"] == 0b11011
    assert hc.hetccl_plan_stages([0, 0, 1, 1], 0, 0)["active"] == 0b11111
    assert hc.hetccl_plan_stages([0, 1, 2, 3], 0, 1)["active"] == 0b110  # RS: B, C
    assert hc.hetccl_plan_stages([0, 1, 2, 3], 0, 2)["active"] == 0b011  # AG: A, B


@pytest.mark.parametrize("name", ["2+2", "1+3", "4+4", "2+6", "2+2+4"])
def test_reduce_bytes(hc, name, unbalanced):
    """Reduce: the root receives every final piece it does not own ((n-1)/n of S for equal pieces), each
    non-root sends its own final pieces; intra/cross bytes as All-Reduce's reduce-scatter half."""
    m = SPLITS[name]
    n = len(m)
    tile = hc.hetccl_plan_info(m, 0, hc.OP_REDUCE, 1 << 28, hc.BFLOAT16)["tile_elems"]
    count = tile * 64
    S = count * 2
    root = n - 1
    ar = [hc.hetccl_plan_info(m, r, hc.OP_ALLREDUCE, count, hc.BFLOAT16) for r in range(n)]
    rd = [hc.hetccl_plan_info(m, r, hc.OP_REDUCE, count, hc.BFLOAT16, root=root) for r in range(n)]
    # the root receives everything but its own pieces
    own_root = S - (rd[root]["bytes_recv"] - ar[root]["bytes_recv"] // 2)
    assert 0 < own_root < S
    assert sum(r["bytes_sent"] for r in rd) == sum(r["bytes_recv"] for r in rd)


def test_all_to_all_bytes(hc):
    for m in ([0, 1], [0, 0, 1, 1], [0] * 4 + [1] * 4):
        n = len(m)
        info = hc.hetccl_plan_info(m, 1, hc.OP_ALL_TO_ALL, 4096, hc.BFLOAT16)
        assert info["bytes_sent"] == info["bytes_recv"] == (n - 1) * 4096 * 2


def test_balanced_tiles(hc):
    """Every channel gets the same number of tiles when the message needs more than one per channel, and
    every piece boundary stays 256-byte aligned."""
    for m in ([0, 1], [0, 0, 1, 1], [0, 1, 2, 2]):
        for mib in (64, 256, 1000):
            i = hc.hetccl_plan_info(m, 0, hc.OP_ALLREDUCE, mib << 19, hc.BFLOAT16)
            k = -(-i["ntiles"] // i["nchannels"])
            assert i["ntiles"] > (k - 1) * i["nchannels"]  # no channel idles for a whole extra tile round
            assert i["ntiles"] <= k * i["nchannels"]
            D = max(m) + 1
            L = 1
            for q in range(D):
                L = L * m.count(q) // __import__("math").gcd(L, m.count(q))
            assert (i["tile_elems"] * 2) % (256 * L * D) == 0  # bf16 pieces of tile/(L*D) are 256-B multiples
