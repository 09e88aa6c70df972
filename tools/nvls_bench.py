"""NVLS mode vs the P2P path, one process driving N GPUs (hetccl_comm_init_all), bf16 sum All-Reduce.

python tools/nvls_bench.py [--gpus 4] [--maps 4,2+2] [--mibs 16,64,256] [--iters 20]
Prints one JSON line per (map, size, mode): busBW = S * 2(n-1)/n / t, t = max over devices of the mean
per-op time (CUDA events on each device's stream, all devices launched back to back every iteration).
Modes: p2p (HETCCL_NVLS unset), nvls (copies in/out of the multicast-bound buffer, 16-bit staged in fp32),
nvls_native16 (same with the switch's native 16-bit adds, HETCCL_NVLS_WIDE=0), nvls_zc (native, in place on
that buffer). Correctness: the R7 gate on rank 0's result against an fp64 sum of sampled windows.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
MAPS = {"2": [0, 0], "1+1": [0, 1], "4": [0, 0, 0, 0], "2+2": [0, 0, 1, 1]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--maps", default="4,2+2")
    ap.add_argument("--mibs", default="16,64,256")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch
    import paper_2601_22585_b200 as hc
    mibs = [int(v) for v in args.mibs.split(",")]
    for name in args.maps.split(","):
        m = MAPS[name]
        n = len(m)
        if n > torch.cuda.device_count():
            continue
        for mode in ("p2p", "nvls", "nvls_native16", "nvls_zc"):
            if mode == "p2p":
                os.environ.pop("HETCCL_NVLS", None)
            else:
                os.environ["HETCCL_NVLS"] = "1"
                os.environ["HETCCL_NVLS_MB"] = str(max(mibs) if mode == "nvls_zc" else 32)
                # nvls: 16-bit staged in fp32 (default, R7 gate); native16 / zc: the switch's own bf16 adds
                # (HETCCL_NVLS_WIDE=0; not RNE, outside the parity bar - DESIGN.md R21)
                os.environ["HETCCL_NVLS_WIDE"] = "1" if mode == "nvls" else "0"
            comms = hc.hetccl_comm_init_all(list(range(n)), m)
            on = hc.hetccl_comm_nvls(comms[0])[0]
            if mode != "p2p" and not on:
                print(json.dumps({"map": name, "mode": mode, "unavailable": str(hc.lib().hetccl_get_last_error(comms[0]))}))
                for c in comms:
                    hc.hetccl_comm_destroy(c)
                continue
            streams = [torch.cuda.Stream(device=r) for r in range(n)]
            for mib in mibs:
                count = mib * (1 << 20) // 2
                g = torch.Generator().manual_seed(7)
                xs_cpu = [(torch.randn(count, generator=g) * 0.0625).bfloat16() for _ in range(n)]
                if mode == "nvls_zc":
                    xs = [hc.nvls_buffer(comms[r], count, torch.bfloat16, r) for r in range(n)]
                    ys = xs
                else:
                    xs = [xs_cpu[r].to(f"cuda:{r}") for r in range(n)]
                    ys = [torch.empty_like(x) for x in xs]
                def run_once():
                    for r in range(n):
                        with torch.cuda.device(r):
                            hc.allreduce(xs[r], ys[r], comms[r], stream=streams[r])
                # correctness on fresh inputs (zero copy: the buffer holds the inputs)
                for r in range(n):
                    xs[r].copy_(xs_cpu[r].to(f"cuda:{r}"))
                for r in range(n):
                    torch.cuda.synchronize(r)
                run_once()
                for r in range(n):
                    torch.cuda.synchronize(r)
                F = np.stack([xs_cpu[r][:65536].float().double().numpy() for r in range(n)])
                R, A = F.sum(0), np.abs(F).sum(0)
                got = ys[0][:65536].float().cpu().double().numpy()
                ok = bool(np.all(np.abs(got - R) <= 1e-2 * A + 1e-30))
                for _ in range(3):
                    run_once()
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
                for r in range(n):
                    torch.cuda.synchronize(r)
                for r in range(n):
                    ev[r][0].record(streams[r])
                for _ in range(args.iters):
                    run_once()
                for r in range(n):
                    ev[r][1].record(streams[r])
                for r in range(n):
                    torch.cuda.synchronize(r)
                t = max(ev[r][0].elapsed_time(ev[r][1]) for r in range(n)) / 1e3 / args.iters
                S = count * 2
                print(json.dumps({"map": name, "n": n, "mode": mode, "mib": mib, "ms": round(t * 1e3, 4),
                                  "busbw": round(S * 2 * (n - 1) / n / t / 1e9, 2), "r7_gate": ok}), flush=True)
                del xs, ys
            for c in comms:
                hc.hetccl_comm_destroy(c)


if __name__ == "__main__":
    main()
