"""Rounding of the NVSwitch reduction (multimem.ld_reduce) in NVLS mode: map "2" (one domain of two GPUs),
random pairs; the two-operand sum is exact in fp64, so each result shows the switch's rounding.
Prints, per dtype, the fraction of results equal to round-to-nearest-even and to round-toward-zero."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["HETCCL_NVLS"] = "1"


def main():
    import torch
    import paper_2601_22585_b200 as hc
    comms = hc.hetccl_comm_init_all([0, 1], [0, 0])
    on = hc.hetccl_comm_nvls(comms[0])[0]
    g = torch.Generator().manual_seed(1)
    n = 1 << 20
    for name, dt in (("bf16", torch.bfloat16), ("f16", torch.float16), ("f32", torch.float32)):
        a = (torch.randn(n, generator=g) * 0.1).to(dt)
        b = (torch.randn(n, generator=g) * 0.01).to(dt)
        xs = [a.to("cuda:0"), b.to("cuda:1")]
        ys = [torch.empty_like(xs[0]), torch.empty_like(xs[1])]
        for r in range(2):
            with torch.cuda.device(r):
                hc.allreduce(xs[r], ys[r], comms[r])
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        got = ys[0].cpu()
        exact = a.double() + b.double()
        rn = exact.to(dt)                       # torch: round to nearest even
        if dt == torch.float32:
            rz = torch.from_numpy(np.nextafter(rn.numpy(), 0).astype(np.float32))
            rz = torch.where((rn.double().abs() > exact.abs()), rz, rn)
        else:  # sign-magnitude: one step toward zero = magnitude bits - 1
            up = rn.double().abs() > exact.abs()
            rz = torch.where(up, (rn.view(torch.int16) - 1).view(dt), rn)
        eq = lambda u, v: (u.view(torch.int16 if dt != torch.float32 else torch.int32) ==
                           v.view(torch.int16 if dt != torch.float32 else torch.int32)).double().mean().item()
        print(json.dumps({"dtype": name, "nvls": on, "n": n, "frac_rne": round(eq(got, rn), 6),
                          "frac_rz": round(eq(got, rz), 6), "rank1_equal": bool(torch.equal(got, ys[1].cpu()))}), flush=True)
    for c in comms:
        hc.hetccl_comm_destroy(c)


if __name__ == "__main__":
    main()
