"""Shared test helpers: seeded inputs (synth), GPU runs through the C ABI binding, comparisons
against the oracle. Imports the oracle (allowed: tests/ only)."""
import numpy as np

import oracle
import synth

MAPS = {
    "1+1": [0, 1], "2": [0, 0], "2+2": [0, 0, 1, 1], "1+3": [0, 1, 1, 1], "1+1+2": [0, 1, 2, 2],
    "4": [0, 0, 0, 0], "4+4": [0, 0, 0, 0, 1, 1, 1, 1], "2+6": [0, 0, 1, 1, 1, 1, 1, 1],
    "2+2+4": [0, 0, 1, 1, 2, 2, 2, 2], "8": [0] * 8, "singletons4": [0, 1, 2, 3],
    "interleaved": [1, 0, 1, 0, 2, 2], "3+5": [0, 0, 0, 1, 1, 1, 1, 1], "1+2+3": [0, 1, 1, 2, 2, 2],
}

TORCH_DT = None


def torch_dtype(dt):
    import torch
    return {"int32": torch.int32, "f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[dt]


def to_torch(a, dt, device):
    """numpy (oracle representation) -> torch tensor of the real dtype on device."""
    import torch
    if dt == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).to(device)
    return torch.from_numpy(a.copy()).to(device)


def to_numpy(t, dt):
    import torch
    t = t.detach().cpu()
    if dt == "bf16":
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    return t.numpy().copy()


def inputs(kind, seed, n, count, dt):
    if kind == "bits" and dt != "int32":
        kind = "normal"
    return [synth.make(kind, seed, r, count, dt) for r in range(n)]


def as_f64(a, dt):
    if dt == "bf16":
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def assert_matches(got, want, xs, dt, op, what=""):
    """The parity bar: bit-exact for int32, f32 and min/max; bf16/f16 sums within the
    north_star gate vs an fp64 reference (normwise <= 1e-2 and elementwise <= 1e-2 * sum|x|) — and,
    since the kernels implement the oracle's rounding points, bit-exact against the oracle too."""
    if dt in ("bf16", "f16") and op == "sum":
        F = np.stack([as_f64(x, dt) for x in xs])
        R = F.sum(0)
        A = np.abs(F).sum(0)
        g = as_f64(got, dt)
        fin = np.isfinite(R)
        err = np.abs(g - R)[fin]
        assert np.all(err <= 1e-2 * A[fin] + 1e-30), f"{what}: elementwise gate failed"
        nrm = np.linalg.norm(R[fin])
        if nrm > 0:
            assert np.linalg.norm(g[fin] - R[fin]) / nrm <= 1e-2, f"{what}: normwise gate failed"
    gb, wb = got.view(np.uint8), want.view(np.uint8)
    if not np.array_equal(gb, wb):
        bad = np.nonzero(got.view(np.uint16 if got.itemsize == 2 else np.uint32) !=
                         want.view(np.uint16 if want.itemsize == 2 else np.uint32))[0]
        raise AssertionError(f"{what}: {bad.size} of {got.size} elements differ from the oracle; first at "
                             f"{bad[:8].tolist()} got {got[bad[:4]]} want {want[bad[:4]]}")
