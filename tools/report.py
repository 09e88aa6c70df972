"""Measurement report for SURVEY §8(d) (one JSON line per row), run under torchrun (one rank per GPU).

  torchrun --nproc-per-node N tools/report.py --what ar_sweep|collectives|c4|c5|splits [--out FILE]

* ar_sweep    : bf16 AR 1 MiB .. 1 GiB (C2), hetccl vs flat NCCL on the same buffers, at the split of N
* splits      : bf16 AR 256 MiB at every split of N GPUs (1+1; 2+2, 1+3, 1+1+2, 4, singletons)
* collectives : bf16 RS / AG / Broadcast / Reduce / All-to-All at 256 MiB (C3 analogue), hetccl vs NCCL
* c4          : 1.3e9-element gradients in 25 MiB buckets, issued round-robin on 1/2/4 streams (one comm per
                stream), wall time per step vs NCCL
* c5          : Llama-7B gradients (6,738,415,616 elements, 13.5 GB bf16 per rank) in 256 MiB buckets
* channels    : AR 256 MiB at the default split with 16 / 32 / 64 / 148 / 296 CTAs per GPU (SM budget) vs NCCL
* overlap     : 24 x 25 MiB buckets all-reduced on a comm stream beside a bf16 GEMM stream: overlap ratio
                (t_gemm + t_comm - t_both) / min, NCCL and hetccl at 64 / 296 CTAs
Times: CUDA events on the launching stream, max over ranks (R16). busBW per R15. Parity: each
measured AR/RS buffer passes DESIGN.md R7's gate vs an fp64 sum on sampled windows (tests/ owns bitwise
parity against the oracle); AG/Broadcast results are compared bitwise with NCCL's.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SPLITS = {2: {"1+1": [0, 1], "2": [0, 0]},
          4: {"2+2": [0, 0, 1, 1], "1+3": [0, 1, 1, 1], "1+1+2": [0, 1, 2, 2], "4": [0, 0, 0, 0],
              "1+1+1+1": [0, 1, 2, 3]},
          8: {"4+4": [0] * 4 + [1] * 4, "2+6": [0, 0] + [1] * 6, "2+2+4": [0, 0, 1, 1, 2, 2, 2, 2]}}
DEFAULT = {2: "1+1", 4: "2+2", 8: "4+4"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="ar_sweep")
    ap.add_argument("--out", default=None)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--split", default=None, help="ar_sweep split (default: 1+1 / 2+2 / 4+4 by world size)")
    ap.add_argument("--mibs", default="1,2,4,8,16,32,64,128,256,512,1024", help="ar_sweep sizes (MiB per rank)")
    ap.add_argument("--kibs", default=None, help="ar_sweep sizes in KiB per rank (overrides --mibs; 1 KiB - 1 MiB "
                                                 "is the latency regime, NEXT-3)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    import paper_2601_22585_b200 as hc
    import synth
    from bench import fp64_gate
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    gloo = dist.new_group(backend="gloo")
    out = open(args.out, "a") if (args.out and rank == 0) else None
    comms = {}

    def comm_for(name, m, slot=0, nch=None):
        key = (name, slot, nch)
        if key not in comms:
            old = os.environ.get("HETCCL_NCHANNELS")
            if nch:
                os.environ["HETCCL_NCHANNELS"] = str(nch)
            comms[key] = hc.init_process_group_comm(m, group=gloo)
            if nch:
                if old is None:
                    del os.environ["HETCCL_NCHANNELS"]
                else:
                    os.environ["HETCCL_NCHANNELS"] = old
        return comms[key]

    def emit(row):
        if rank == 0:
            line = json.dumps(row)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
                out.flush()

    def timed(fn, iters, warm=3, stream=None, graph=False):
        """Mean device time per call (CUDA events, max over ranks). graph=True captures the `iters` calls
        in one CUDA graph first, so host launch overhead does not bound small messages."""
        s = stream or torch.cuda.current_stream()
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        g = None
        if graph:
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                with torch.cuda.graph(g, stream=cs):
                    for _ in range(iters):
                        fn()
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        if g is not None:
            g.replay()
        else:
            for _ in range(iters):
                fn()
        b.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / iters], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item() * 1e-3

    def bf16_inputs(seed, count):
        x = synth.normal(seed, rank, count, "bf16")
        return torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to("cuda")

    def parity_ar(y, seed, count, m):
        W = 2048
        ok = True
        for st in (0, max(0, count // 2 - W // 2), max(0, count - W)):
            w = min(W, count - st)
            xs = [synth.normal(seed, r, w, "bf16", start=st) for r in range(world)]
            got = y[st:st + w].cpu().view(torch.int16).numpy().view(np.uint16)
            ok &= fp64_gate(got, xs)
        t = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    def ar_row(name, m, mib, seed=2, iters=None, kib=None):
        count = (kib * 1024 if kib is not None else mib * (1 << 20)) // 2
        S = count * 2
        mib = S / (1 << 20)
        x = bf16_inputs(seed, count)
        y = torch.empty_like(x)
        c = comm_for(name, m)
        it = iters or (args.iters if mib <= 256 else max(3, args.iters // 4))
        graph = mib <= 16  # launch-latency regime: time CUDA-graph replays (both libraries)
        if graph:
            it = 50
        t_staged = timed(lambda: hc.allreduce(x, y, c), it, graph=graph)
        ok = parity_ar(y, seed, count, m)
        # symmetric send + recv buffers (hetccl_mem_*): peers' x read directly (pull), results written
        # straight into the peers' buffers (direct)
        xsym = hc.symmetric_empty(c, count, torch.bfloat16, group=gloo)
        xsym.copy_(x)
        ysym = hc.symmetric_empty(c, count, torch.bfloat16, group=gloo)
        t = timed(lambda: hc.allreduce(xsym, ysym, c), it, graph=graph)
        ok = ok and parity_ar(ysym, seed, count, m)
        hc.lib().hetccl_mem_free(c, ysym.data_ptr())
        hc.lib().hetccl_mem_free(c, xsym.data_ptr())
        del ysym, xsym
        z = x.clone()
        tn = timed(lambda: dist.all_reduce(z), it, graph=graph)
        alg = S / t / 1e9
        bus = alg * 2 * (world - 1) / world
        nbus = S / tn / 1e9 * 2 * (world - 1) / world
        busiest = max(hc.hetccl_plan_info(m, r, hc.OP_ALLREDUCE, count, hc.BFLOAT16)["bytes_sent"] for r in range(world))
        emit({"row": "allreduce", "split": name, "map": m, "n": world, "bytes": S, "dtype": "bf16", "ms": round(t * 1e3, 4),
              "algbw": round(alg, 2), "busbw": round(bus, 2), "nccl_busbw": round(nbus, 2),
              "vs_nccl": round(bus / nbus, 4), "busbw_over_900": round(bus / 900, 4),
              "link_util_770": round(busiest / t / 1e9 / 770, 4), "r7_gate": ok, "cuda_graph": graph,
              "staged_busbw": round(S / t_staged / 1e9 * 2 * (world - 1) / world, 2),
              "us": round(t * 1e6, 2), "nccl_us": round(tn * 1e6, 2), "staged_us": round(t_staged * 1e6, 2),
              "note": "busbw: send/recv in symmetric buffers (pull + direct); staged_busbw: plain torch buffers"})
        del x, y, z

    if args.what == "ar_sweep":
        name = args.split or DEFAULT[world]
        m = SPLITS[world][name]
        if args.kibs:
            for kib in [int(v) for v in args.kibs.split(",")]:
                ar_row(name, m, None, kib=kib)
        else:
            for mib in [int(v) for v in args.mibs.split(",")]:
                ar_row(name, m, mib)
    elif args.what == "splits":
        for name, m in SPLITS[world].items():
            ar_row(name, m, 256)
    elif args.what == "collectives":
        for name, m in SPLITS[world].items():
            if world == 4 and name not in ("2+2", "1+3", "1+1+2"):
                continue
            c = comm_for(name, m)
            S = 256 << 20
            count = S // 2
            R = count // world
            x = bf16_inputs(3, count)
            # reduce-scatter
            y = torch.empty(R, dtype=torch.bfloat16, device="cuda")
            t = timed(lambda: hc.reduce_scatter(x, y, c), args.iters)
            W = 2048
            ok = True
            if rank == 0:  # my block = elements [0, R) of every rank's input
                got = y.cpu().view(torch.int16).numpy().view(np.uint16)
                for st in (0, R - W):
                    xs = [synth.normal(3, r, W, "bf16", start=st) for r in range(world)]
                    ok &= fp64_gate(got[st:st + W], xs)
            yn = torch.empty_like(y)
            tn = timed(lambda: dist.reduce_scatter_tensor(yn, x), args.iters)
            f = (world - 1) / world
            emit({"row": "reduce_scatter", "split": name, "n": world, "bytes": S, "ms": round(t * 1e3, 4),
                  "busbw": round(S / t / 1e9 * f, 2), "nccl_busbw": round(S / tn / 1e9 * f, 2),
                  "vs_nccl": round(tn / t, 4), "r7_gate_rank0": ok})
            # all-gather
            xa = x[:R].contiguous()
            ya = torch.empty(count, dtype=torch.bfloat16, device="cuda")
            t = timed(lambda: hc.all_gather(xa, ya, c), args.iters)
            yn = torch.empty_like(ya)
            tn = timed(lambda: dist.all_gather_into_tensor(yn, xa), args.iters)
            ok = bool(torch.equal(ya.view(torch.int16), yn.view(torch.int16)))
            emit({"row": "all_gather", "split": name, "n": world, "bytes": S, "ms": round(t * 1e3, 4),
                  "busbw": round(S / t / 1e9 * f, 2), "nccl_busbw": round(S / tn / 1e9 * f, 2),
                  "vs_nccl": round(tn / t, 4), "equals_nccl_bitwise": ok})
            # broadcast (root = last rank)
            yb = torch.empty_like(x)
            root = world - 1
            t = timed(lambda: hc.broadcast(x, yb, root, c), args.iters)
            zb = x.clone()
            tn = timed(lambda: dist.broadcast(zb, src=root), args.iters)
            ok = bool(torch.equal(yb.view(torch.int16), zb.view(torch.int16)))
            emit({"row": "broadcast", "split": name, "n": world, "bytes": S, "ms": round(t * 1e3, 4),
                  "busbw": round(S / t / 1e9, 2), "nccl_busbw": round(S / tn / 1e9, 2), "vs_nccl": round(tn / t, 4),
                  "equals_nccl_bitwise": ok})
            # reduce (root = last rank) and all-to-all (NEXT-2)
            yr = torch.empty_like(x) if rank == root else None
            t = timed(lambda: hc.reduce(x, yr, root, c), args.iters)
            zr = x.clone()
            tn = timed(lambda: dist.reduce(zr, dst=root), args.iters)
            emit({"row": "reduce", "split": name, "n": world, "bytes": S, "ms": round(t * 1e3, 4),
                  "busbw": round(S / t / 1e9, 2), "nccl_busbw": round(S / tn / 1e9, 2), "vs_nccl": round(tn / t, 4)})
            y2 = torch.empty_like(x)
            t = timed(lambda: hc.all_to_all(x, y2, c), args.iters)
            z2 = torch.empty_like(x)
            tn = timed(lambda: dist.all_to_all_single(z2, x), args.iters)
            ok = bool(torch.equal(y2.view(torch.int16), z2.view(torch.int16)))
            emit({"row": "all_to_all", "split": name, "n": world, "bytes": S, "ms": round(t * 1e3, 4),
                  "busbw": round(S / t / 1e9 * f, 2), "nccl_busbw": round(S / tn / 1e9 * f, 2),
                  "vs_nccl": round(tn / t, 4), "equals_nccl_bitwise": ok})
            del x, y, ya, yb, yn, zb, yr, zr, y2, z2
    elif args.what == "channels":
        # SM budget: AR 256 MiB at the default split on symmetric buffers with 16..296 CTAs per GPU
        name = DEFAULT[world]
        m = SPLITS[world][name]
        count = 128 << 20
        x = bf16_inputs(2, count)
        z = x.clone()
        tn = timed(lambda: dist.all_reduce(z), args.iters)
        nbus = count * 2 / tn / 1e9 * 2 * (world - 1) / world
        for nch in (16, 32, 64, 148, 296):
            c = comm_for(name, m, slot=100 + nch, nch=nch)
            xs = hc.symmetric_empty(c, count, torch.bfloat16, group=gloo)
            ys = hc.symmetric_empty(c, count, torch.bfloat16, group=gloo)
            xs.copy_(x)
            t = timed(lambda: hc.allreduce(xs, ys, c), args.iters)
            ok = parity_ar(ys, 2, count, m)
            bus = count * 2 / t / 1e9 * 2 * (world - 1) / world
            emit({"row": "channels", "split": name, "n": world, "ctas_per_gpu": nch, "bytes": count * 2,
                  "ms": round(t * 1e3, 4), "busbw": round(bus, 2), "nccl_busbw": round(nbus, 2),
                  "vs_nccl": round(bus / nbus, 4), "r7_gate": ok})
            hc.lib().hetccl_mem_free(c, ys.data_ptr())
            hc.lib().hetccl_mem_free(c, xs.data_ptr())
    elif args.what == "overlap":
        # C4-style gradient buckets all-reduced on a comm stream while a bf16 GEMM stream runs:
        # overlap = (t_gemm + t_comm - t_both) / min(t_gemm, t_comm), 1 = fully hidden, 0 = serialised
        name = {2: "1+1", 4: "1+1+2", 8: "2+2+4"}[world]
        m = SPLITS[world][name]
        nb, bucket = 24, 25 * (1 << 20) // 2
        g = bf16_inputs(4, nb * bucket)
        A = torch.randn(8192, 8192, device="cuda").bfloat16()
        B = torch.randn(8192, 8192, device="cuda").bfloat16()
        C = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
        sg, sc = torch.cuda.Stream(), torch.cuda.Stream()
        cur = torch.cuda.current_stream()

        def gemm():
            sg.wait_stream(cur)
            with torch.cuda.stream(sg):
                for _ in range(8):
                    torch.matmul(A, B, out=C)
            cur.wait_stream(sg)

        def run(comm_fn, with_gemm):
            def step():
                sc.wait_stream(cur)
                if with_gemm:
                    sg.wait_stream(cur)
                    with torch.cuda.stream(sg):
                        for _ in range(8):
                            torch.matmul(A, B, out=C)
                with torch.cuda.stream(sc):
                    comm_fn()
                cur.wait_stream(sc)
                if with_gemm:
                    cur.wait_stream(sg)
            return timed(step, 3, warm=1)
        t_gemm = timed(gemm, 3, warm=1)
        red = g.clone()

        def nccl_fn():
            for b in range(nb):
                dist.all_reduce(red[b * bucket:(b + 1) * bucket])
        rows = [("nccl", nccl_fn)]
        for nch in (64, 296):
            c = comm_for(name, m, slot=200 + nch, nch=nch)

            def hc_fn(c=c):
                for b in range(nb):
                    hc.hetccl_allreduce(g[b * bucket:].data_ptr(), red[b * bucket:].data_ptr(), bucket, hc.BFLOAT16,
                                        "sum", c, sc.cuda_stream)
            rows.append((f"hetccl_{nch}ch", hc_fn))
        for label, fn in rows:
            t_comm = run(fn, False)
            t_both = run(fn, True)
            emit({"row": "overlap", "split": name, "n": world, "impl": label, "buckets": nb,
                  "bytes": nb * bucket * 2, "gemm_ms": round(t_gemm * 1e3, 3), "comm_ms": round(t_comm * 1e3, 3),
                  "both_ms": round(t_both * 1e3, 3),
                  "overlap": round((t_gemm + t_comm - t_both) / min(t_gemm, t_comm), 4),
                  "comm_busbw": round(nb * bucket * 2 / t_comm / 1e9 * 2 * (world - 1) / world, 2)})
    elif args.what == "c4":
        name = {2: "1+1", 4: "1+1+2", 8: "2+2+4"}[world]
        m = SPLITS[world][name]
        total = 1_300_000_000
        bucket = 25 * (1 << 20) // 2
        sizes = [bucket] * (total // bucket) + ([total % bucket] if total % bucket else [])
        g = bf16_inputs(4, total)
        # the reduced-gradient buffer is symmetric (hetccl_mem_*), one per stream comm set: results land
        # straight in the peers' buffers; comms of every stream count connect to the first one's buffer
        out_g = None
        offs = np.cumsum([0] + sizes)
        for nstreams in (1, 2, 4):
            streams = [torch.cuda.Stream() for _ in range(nstreams)]
            # concurrent persistent kernels must be co-resident: split the SMs between the streams' comms
            slots = 592 if os.environ.get("HETCCL_LEGACY") == "0" else 296  # CTAs per GPU of the kernel build
            cs = [comm_for(name, m, slot=i, nch=slots // nstreams) for i in range(nstreams)]
            outs = [hc.symmetric_empty(c, total, torch.bfloat16, group=gloo) for c in cs]
            out_g = outs[0]
            cur = torch.cuda.current_stream()

            def step():
                for s in streams:
                    s.wait_stream(cur)
                for b, sz in enumerate(sizes):
                    i = b % nstreams
                    hc.hetccl_allreduce(g[offs[b]:].data_ptr(), outs[i][offs[b]:].data_ptr(), int(sz), hc.BFLOAT16,
                                        "sum", cs[i], streams[i].cuda_stream)
                for s in streams:
                    cur.wait_stream(s)
            t = timed(step, 3, warm=1)
            if nstreams > 1:  # bucket b was reduced into outs[b % nstreams]; gather the result into out_g
                for b, sz in enumerate(sizes):
                    if b % nstreams:
                        out_g[offs[b]:offs[b] + sz].copy_(outs[b % nstreams][offs[b]:offs[b] + sz])
            for c, o in zip(cs[1:], outs[1:]):
                hc.lib().hetccl_mem_free(c, o.data_ptr())
            emit({"row": "c4_buckets", "split": name, "n": world, "streams": nstreams, "buckets": len(sizes),
                  "bytes": total * 2, "ms": round(t * 1e3, 3),
                  "eff_busbw": round(total * 2 / t / 1e9 * 2 * (world - 1) / world, 2)})
        ok = parity_ar(out_g, 4, total, m)
        z = g.clone()

        def nstep():
            for b, sz in enumerate(sizes):
                dist.all_reduce(z[offs[b]:offs[b] + sz])
        tn = timed(nstep, 3, warm=1)
        emit({"row": "c4_buckets_nccl", "split": "flat", "n": world, "buckets": len(sizes), "bytes": total * 2,
              "ms": round(tn * 1e3, 3), "eff_busbw": round(total * 2 / tn / 1e9 * 2 * (world - 1) / world, 2),
              "hetccl_r7_gate": ok})
    elif args.what == "c5":
        name = DEFAULT[world]
        m = SPLITS[world][name]
        total = 6_738_415_616
        bucket = 256 * (1 << 20) // 2
        sizes = [bucket] * (total // bucket) + ([total % bucket] if total % bucket else [])
        c = comm_for(name, m)
        g = hc.symmetric_empty(c, total, torch.bfloat16, group=gloo)  # the gradient buffer is symmetric
        g.normal_(0, 1.0 / 16, generator=torch.Generator("cuda").manual_seed(5 + rank))
        offs = np.cumsum([0] + sizes)

        def step():
            for b, sz in enumerate(sizes):
                p = g[offs[b]:].data_ptr()
                hc.hetccl_allreduce(p, p, int(sz), hc.BFLOAT16, "sum", c, torch.cuda.current_stream().cuda_stream)
        t = timed(step, 2, warm=1)

        def nstep():
            for b, sz in enumerate(sizes):
                dist.all_reduce(g[offs[b]:offs[b] + sz])
        tn = timed(nstep, 2, warm=1)
        S = total * 2
        emit({"row": "c5_llama7b", "split": name, "n": world, "buckets": len(sizes), "bytes": S, "ms": round(t * 1e3, 2),
              "eff_busbw": round(S / t / 1e9 * 2 * (world - 1) / world, 2), "nccl_ms": round(tn * 1e3, 2),
              "nccl_eff_busbw": round(S / tn / 1e9 * 2 * (world - 1) / world, 2), "vs_nccl": round(tn / t, 4),
              "note": "in-place; values grow across repeated steps (timing only; parity in tests)"})
    for c in comms.values():
        hc.hetccl_comm_destroy(c)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
