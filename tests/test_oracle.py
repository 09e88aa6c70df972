"""Pins for the CPU oracle (tests -m "not gpu"). Each check ties the oracle to something other than
itself: the paper/SPEC worked examples (tests/golden/, cited per fixture), hand-derived values,
closed forms, textbook special cases (plain left folds in numpy scalar arithmetic), invariants,
brute force on tiny inputs, an independent library's conversions, and floating-point error bounds.
"""
import itertools
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _arr(vals, dtype):
    if dtype == "bf16":
        return (np.asarray(vals, np.float32).view(np.uint32) >> 16).astype(np.uint16)
    return np.asarray(vals, oracle.NP_DTYPE[oracle.DTYPE_NAMES[dtype]])


def _hex(vals, dtype):
    w = np.uint16 if dtype in ("bf16", "f16") else np.uint32
    a = np.array([int(v, 16) for v in vals], dtype=w)
    return a.view(oracle.NP_DTYPE[oracle.DTYPE_NAMES[dtype]]) if dtype != "bf16" else a


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [json.loads(l) for l in f if l.strip()]


@pytest.mark.parametrize("case", _load("spec_examples.jsonl"), ids=lambda c: c["id"])
def test_spec_worked_examples(case):
    dt = case["dtype"]
    xs = [_arr(x, dt) for x in case["x"]]
    op = case["op"]
    if op == "allreduce":
        y = oracle.allreduce(xs, case["map"], dt, case["red"])
        for want in case["y"]:
            np.testing.assert_array_equal(y, _arr(want, dt))
    elif op == "reduce_scatter":
        ys = oracle.reduce_scatter(xs, case["map"], dt, case["red"])
        for y, want in zip(ys, case["y"]):
            np.testing.assert_array_equal(y, _arr(want, dt))
    elif op == "all_gather":
        for y, want in zip(oracle.all_gather(xs, dt), case["y"]):
            np.testing.assert_array_equal(y, _arr(want, dt))
    elif op == "broadcast":
        for y, want in zip(oracle.broadcast(xs, case["root"], dt), case["y"]):
            np.testing.assert_array_equal(y, _arr(want, dt))
    elif op == "reduce":
        y = oracle.reduce(xs, case["map"], case["root"], dt, case["red"])
        np.testing.assert_array_equal(y, _arr(case["y_root"], dt))
    elif op == "all_to_all":
        for y, want in zip(oracle.all_to_all(xs, dt), case["y"]):
            np.testing.assert_array_equal(y, _arr(want, dt))
    else:
        raise AssertionError(op)


@pytest.mark.parametrize("case", _load("hand_worked.jsonl"), ids=lambda c: c["id"])
def test_hand_worked_examples(case):
    dt = case["dtype"]
    xs = [_hex(x, dt) for x in case["x_hex"]]
    y = oracle.allreduce(xs, case["map"], dt, case["red"])
    want = _hex(case["y_hex"], dt)
    np.testing.assert_array_equal(y.view(want.dtype), want)


MAPS = {
    "1+1": [0, 1], "2": [0, 0], "2+2": [0, 0, 1, 1], "1+3": [0, 1, 1, 1], "1+1+2": [0, 1, 2, 2],
    "4+4": [0, 0, 0, 0, 1, 1, 1, 1], "2+6": [0, 0, 1, 1, 1, 1, 1, 1], "2+2+4": [0, 0, 1, 1, 2, 2, 2, 2],
    "interleaved": [1, 0, 1, 0, 2, 2], "8": [0] * 8, "singletons8": list(range(8)),
}


@pytest.mark.parametrize("name", sorted(MAPS))
@pytest.mark.parametrize("dtype", ["f32", "int32"])
def test_ramp_closed_form(name, dtype):
    """x_r[i] = (i mod M) + M r  =>  Y[i] = n (i mod M) + M n (n-1)/2, exact in f32 below 2^24."""
    m = MAPS[name]
    n, M, count = len(m), 4096, 3 * 4096 + 77
    xs = [synth.ramp(r, count, M, dtype) for r in range(n)]
    y = oracle.allreduce(xs, m, dtype, "sum")
    i = np.arange(count)
    want = n * (i % M) + M * n * (n - 1) // 2
    np.testing.assert_array_equal(y.astype(np.int64), want)


@pytest.mark.parametrize("name", ["4+4", "2+6", "2+2+4", "8", "singletons8"])
def test_bf16_ramp_closed_form(name):
    """bf16: x_r[i] = (i mod 16) + r at n=8 -> all partial and final sums are integers <= 148 (exact)."""
    m = MAPS[name]
    count = 1000
    xs = [synth.ramp(0, count, 16, "f32") + r for r in range(8)]
    xs = [(x.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16) for x in xs]
    y = oracle.allreduce(xs, m, "bf16", "sum")
    yf = (y.astype(np.uint32) << 16).view(np.float32)
    np.testing.assert_array_equal(yf, 8 * (np.arange(count) % 16) + 28)


def _left_fold_f32(cols):
    acc = np.float32(cols[0])
    for v in cols[1:]:
        acc = np.float32(acc + np.float32(v))
    return acc


@pytest.mark.parametrize("m", [[0, 0, 0, 0, 0], [0, 1, 2, 3, 4]])
def test_textbook_left_fold_special_cases(m):
    """D=1 and all-singleton ascending maps reduce to a plain ascending-rank left fold."""
    n, count = len(m), 257
    xs = [synth.uniform(11, r, count, "f32", -1e3, 1e3) for r in range(n)]
    y = oracle.allreduce(xs, m, "f32", "sum")
    want = np.array([_left_fold_f32([x[i] for x in xs]) for i in range(count)], np.float32)
    np.testing.assert_array_equal(y, want)


def test_two_level_fold_by_hand_numpy():
    """2+6 with generic fp32 data: recompute the domain-major fold with numpy float32 scalars."""
    m = MAPS["2+6"]
    count = 129
    xs = [synth.uniform(5, r, count, "f32") for r in range(8)]
    y = oracle.allreduce(xs, m, "f32", "sum")
    for i in range(count):
        p0 = _left_fold_f32([xs[0][i], xs[1][i]])
        p1 = _left_fold_f32([xs[r][i] for r in range(2, 8)])
        assert y[i] == np.float32(p0 + p1)


def test_bf16_staged_by_torch_rounding():
    """bf16 sum recomputed with torch's (independent) f32->bf16 RNE cast at the domain boundary."""
    m = MAPS["2+2+4"]
    count = 4099
    xs = [synth.normal(7, r, count, "bf16") for r in range(8)]
    y = oracle.allreduce(xs, m, "bf16", "sum")
    X = torch.stack([torch.from_numpy(x.astype(np.int32) << 16).view(torch.float32) for x in xs])
    parts = []
    for k in range(3):
        ranks = [r for r in range(8) if m[r] == k]
        a = X[ranks[0]].clone()
        for r in ranks[1:]:
            a = a + X[r]
        parts.append(a.to(torch.bfloat16).to(torch.float32))
    acc = parts[0] + parts[1]
    acc = acc + parts[2]
    want = acc.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(y, want)


def _valid_maps(n):
    for m in itertools.product(range(n), repeat=n):
        D = max(m) + 1
        if set(m) == set(range(D)):
            yield list(m)


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_bruteforce_int32_all_maps(n):
    """Every valid map for n<=4: random int32 (wrapping) -> the plain sum mod 2^32; min/max -> numpy."""
    count = 64
    xs = [synth.bits(3, r, count) for r in range(n)]
    S = np.sum(np.stack(xs).astype(np.int64), axis=0)
    want = ((S + 2**31) % 2**32 - 2**31).astype(np.int32)
    for m in _valid_maps(n):
        np.testing.assert_array_equal(oracle.allreduce(xs, m, "int32", "sum"), want)
        np.testing.assert_array_equal(oracle.allreduce(xs, m, "int32", "max"), np.max(np.stack(xs), 0))
        np.testing.assert_array_equal(oracle.allreduce(xs, m, "int32", "min"), np.min(np.stack(xs), 0))


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_minmax_order_free(dtype):
    """min/max are order-free: equal across maps and equal to numpy's elementwise min/max."""
    count = 333
    xs = [synth.uniform(9, r, count, dtype) for r in range(8)]
    if dtype == "bf16":
        F = np.stack([(x.astype(np.uint32) << 16).view(np.float32) for x in xs])
    else:
        F = np.stack(xs).astype(np.float32)
    for name in ("4+4", "2+6", "2+2+4", "8", "singletons8"):
        mx = oracle.allreduce(xs, MAPS[name], dtype, "max")
        mn = oracle.allreduce(xs, MAPS[name], dtype, "min")
        if dtype == "bf16":
            mx, mn = (mx.astype(np.uint32) << 16).view(np.float32), (mn.astype(np.uint32) << 16).view(np.float32)
        np.testing.assert_array_equal(mx.astype(np.float32), F.max(0))
        np.testing.assert_array_equal(mn.astype(np.float32), F.min(0))


def test_permutation_invariance_int32():
    """Permuting ranks together with their map entries leaves the result unchanged (int32 is exact)."""
    rng = np.random.default_rng(0)
    m = MAPS["2+2+4"]
    xs = [synth.bits(4, r, 500) for r in range(8)]
    base = oracle.allreduce(xs, m, "int32", "sum")
    for _ in range(5):
        p = rng.permutation(8)
        xs_p = [xs[i] for i in p]
        m_p = [m[i] for i in p]
        np.testing.assert_array_equal(oracle.allreduce(xs_p, m_p, "int32", "sum"), base)


def test_split_invariance_exact_data():
    """Any domain split gives the same f32 result when all partial sums are exact (ramp data)."""
    xs = [synth.ramp(r, 1000, 512, "f32") for r in range(8)]
    ref = oracle.allreduce(xs, MAPS["8"], "f32", "sum")
    for name in ("4+4", "2+6", "2+2+4", "singletons8"):
        np.testing.assert_array_equal(oracle.allreduce(xs, MAPS[name], "f32", "sum"), ref)


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16", "int32"])
@pytest.mark.parametrize("name", ["2+6", "1+1+2", "4+4"])
def test_allreduce_equals_allgather_of_reducescatter(dtype, name):
    m = MAPS[name]
    n = len(m)
    xs = [synth.make("bits" if dtype == "int32" else "normal", 6, r, n * 37, dtype) for r in range(n)]
    y = oracle.allreduce(xs, m, dtype, "sum")
    rs = oracle.reduce_scatter(xs, m, dtype, "sum")
    for out in oracle.all_gather(rs, dtype):
        np.testing.assert_array_equal(out.view(np.uint8), y.view(np.uint8))


def test_f32_error_bound():
    """Recursive summation bound |Y - R| <= gamma_{n-1} sum|x| with R the fp64 sum (Higham, Thm 4.1)."""
    for name in ("4+4", "2+6", "2+2+4", "singletons8"):
        xs = [synth.uniform(21, r, 4096, "f32", -1, 1) for r in range(8)]
        y = oracle.allreduce(xs, MAPS[name], "f32", "sum").astype(np.float64)
        X = np.stack(xs).astype(np.float64)
        R = X.sum(0)
        u = 2.0**-24
        g = 7 * u / (1 - 7 * u)
        assert np.all(np.abs(y - R) <= g * np.abs(X).sum(0) + 1e-300)


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_16bit_tolerance_gate(dtype):
    """16-bit sum with staged rounding stays within the north_star gate (reading R7)."""
    u = 2.0**-8 if dtype == "bf16" else 2.0**-11
    for name in ("4+4", "2+6", "2+2+4"):
        xs = [synth.normal(2, r, 1 << 14, dtype) for r in range(8)]
        y = oracle.allreduce(xs, MAPS[name], dtype, "sum")
        if dtype == "bf16":
            F = np.stack([(x.astype(np.uint32) << 16).view(np.float32) for x in xs]).astype(np.float64)
            yf = (y.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        else:
            F = np.stack(xs).astype(np.float64)
            yf = y.astype(np.float64)
        R = F.sum(0)
        A = np.abs(F).sum(0)
        g = 7 * 2.0**-24 / (1 - 7 * 2.0**-24)
        assert np.all(np.abs(yf - R) <= (2 * u + g) * A)
        assert np.linalg.norm(yf - R) / np.linalg.norm(R) <= 1e-2
        assert np.all(np.abs(yf - R) <= 1e-2 * A)


def test_conversions_against_libraries():
    """f32->bf16 RNE vs torch; f32->f16 vs numpy; including ties, NaN, inf and subnormals."""
    special = np.array([0.0, -0.0, 1.0, 1.00390625, 1.01171875, 3.3961e38, -3.4e38, np.inf, -np.inf,
                        1e-45, 1e-40, 6.1e-5, 5.96e-8, 2.98e-8, 65504.0, 65520.0, 1e5], np.float32)
    rnd = synth.uniform(1, 0, 5000, "f32", -1e4, 1e4) * np.float32(1e-3)
    vals = np.concatenate([special, rnd, rnd * np.float32(1e-38)])
    tb = torch.from_numpy(vals).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    ob = np.array([oracle.f32_to_bf16(v) for v in vals], np.uint16)
    np.testing.assert_array_equal(ob, tb)
    nh = vals.astype(np.float16).view(np.uint16)
    oh = np.array([oracle.f32_to_f16(v) for v in vals], np.uint16)
    np.testing.assert_array_equal(oh, nh)
    # NaN -> quiet NaN (class only; payload unpinned, reading R10)
    b = oracle.f32_to_bf16(float("nan"))
    assert (b & 0x7f80) == 0x7f80 and (b & 0x7f) != 0
    # widening is exact
    for h in (0x0001, 0x3c00, 0x7bff, 0x8400):
        assert oracle.f16_to_f32(h) == float(np.array([h], np.uint16).view(np.float16)[0])


@pytest.mark.parametrize("bad", [[1, 1], [0, 2], [-1, 0], [0, 0, 2]])
def test_invalid_maps_rejected(bad):
    xs = [np.zeros(4, np.float32) for _ in bad]
    with pytest.raises(ValueError):
        oracle.allreduce(xs, bad, "f32", "sum")


def test_broadcast_allgather_alltoall_labels():
    n = 5
    xs = [np.arange(6, dtype=np.int32) + 100 * r for r in range(n)]
    for root in range(n):
        for y in oracle.broadcast(xs, root, "int32"):
            np.testing.assert_array_equal(y, xs[root])
    for y in oracle.all_gather(xs, "int32"):
        np.testing.assert_array_equal(y, np.concatenate(xs))
    xs = [np.arange(10, dtype=np.int32) + 100 * r for r in range(n)]  # 2 elems per block
    ys = oracle.all_to_all(xs, "int32")
    for i in range(n):
        np.testing.assert_array_equal(ys[i], np.concatenate([xs[j][2 * i:2 * i + 2] for j in range(n)]))


@pytest.mark.parametrize("dt,op", [("bf16", "sum"), ("f32", "sum"), ("int32", "max"), ("f16", "min")])
@pytest.mark.parametrize("m", [[0, 0, 0, 0, 1, 1, 1, 1], [0, 1, 2, 2], [1, 0, 1, 0, 2, 2]])
def test_threaded_oracle_splits_elements_only(dt, op, m):
    """the T-thread oracle splits elements only, so its Y is bit-identical to the serial one
    (ragged per-thread ranges, more threads than some ranges)."""
    n, count = len(m), 100_003
    kind = "bits" if dt == "int32" else "normal"
    xs = [synth.make(kind, 41, r, count, dt) for r in range(n)]
    want = oracle.allreduce(xs, m, dt, op)
    for T in (1, 3, 7, 16):
        got = oracle.allreduce_threaded(xs, m, dt, op, threads=T)
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), f"T={T}"
