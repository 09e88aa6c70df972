"""Per-iteration phase breakdown of the pipelined kernels (profiling aid, not a benchmark).

torchrun --nproc-per-node N tools/trace_run.py [--mib 256] [--op ar|rs|ag|bc] [--out DIR]
Each rank: one warm-up op, then one op with HETCCL_TRACE_ITERS stamps; saves trace_r{rank}.npy and
prints (rank 0) the mean per-iteration time split into wait / work / fence and the kernel span.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("HETCCL_TRACE_ITERS", "256")

MAPS = {2: [0, 1], 4: [0, 0, 1, 1], 8: [0, 0, 0, 0, 1, 1, 1, 1]}


def summarize(tr, label):
    # tr: [rows, ch, it, 4]
    rows, nch, iters, _ = tr.shape
    used = tr[..., 0] > 0
    t0 = tr[..., 0][used].min()
    t_end = tr[..., 3][used].max()
    wait = (tr[..., 1] - tr[..., 0]).astype(np.int64)[used]
    work = (tr[..., 2] - tr[..., 1]).astype(np.int64)[used]
    fence = (tr[..., 3] - tr[..., 2]).astype(np.int64)[used]
    nit = used.sum(axis=2)
    if tr.shape[-1] >= 10:
        ent, ext = tr[..., 0, 8].astype(np.int64), tr[..., 0, 9].astype(np.int64)
        e0 = ent[ent > 0].min()
        print(f"{label}: kernel entry spread {(ent.max() - e0) / 1e3:.1f} us, first poll {(t0 - e0) / 1e3:.1f} us after "
              f"the first entry, exits {(ext[ext > 0].min() - e0) / 1e3:.1f}..{(ext.max() - e0) / 1e3:.1f} us")
    print(f"{label}: span {(t_end - t0) / 1e3:.1f} us, iterations/channel {nit.min()}..{nit.max()}, "
          f"per iteration mean wait {wait.mean() / 1e3:.2f} us, work {work.mean() / 1e3:.2f} us, "
          f"fence {fence.mean() / 1e3:.2f} us; p90 wait {np.percentile(wait, 90) / 1e3:.2f} "
          f"work {np.percentile(work, 90) / 1e3:.2f} fence {np.percentile(fence, 90) / 1e3:.2f}")
    # per logical stage: time from the previous stamp (work start or the previous stage's end)
    st = tr[..., 4:8].astype(np.int64)
    prev = tr[..., 1].astype(np.int64)
    names = "ABCD"
    parts = []
    for s in range(4):
        m = used & (st[..., s] > 0)
        if m.any():
            parts.append(f"{names[s]} {(st[..., s] - prev)[m].mean() / 1e3:.2f}")
            prev = np.where(st[..., s] > 0, st[..., s], prev)
    tail = (tr[..., 2].astype(np.int64) - prev)[used]
    print("  per stage (us, mean over iterations where it ran): " + ", ".join(parts) + f", E/rest {tail.mean() / 1e3:.2f}")
    # by iteration index (mean over channels/rows)
    for it in list(range(min(6, iters))) + [iters // 2]:
        m = used[..., it]
        if not m.any():
            continue
        print(f"  it {it:3d}: wait {(tr[..., it, 1] - tr[..., it, 0])[m].astype(np.int64).mean() / 1e3:7.2f}  "
              f"work {(tr[..., it, 2] - tr[..., it, 1])[m].astype(np.int64).mean() / 1e3:7.2f}  "
              f"fence {(tr[..., it, 3] - tr[..., it, 2])[m].astype(np.int64).mean() / 1e3:7.2f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--op", default="ar")
    ap.add_argument("--out", default="gpurun_out/trace")
    ap.add_argument("--sym", action="store_true", help="All-Reduce into a symmetric buffer (direct path)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    import paper_2601_22585_b200 as hc
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    os.makedirs(args.out, exist_ok=True)
    if world == 1:  # mux 4+4 on one GPU
        m = MAPS[8]
        n = len(m)
        count = args.mib * (1 << 20) // 2
        xs = [torch.randn(count, device="cuda").bfloat16() for _ in range(n)]
        ys = [torch.empty_like(x) for x in xs]
        comm = hc.hetccl_comm_init_mux(n, m, 0)
        for _ in range(2):
            hc.mux_allreduce(xs, ys, comm)
        torch.cuda.synchronize()
        tr = hc.hetccl_comm_get_trace(comm)
        np.save(os.path.join(args.out, "trace_mux.npy"), tr)
        summarize(tr, f"mux 4+4 AR {args.mib} MiB")
        return
    dist.init_process_group("gloo")
    m = MAPS[world]
    comm = hc.init_process_group_comm(m)
    count = args.mib * (1 << 20) // 2
    x = torch.randn(count, device="cuda").bfloat16()
    if args.op == "ar":
        y = hc.symmetric_empty(comm, count, torch.bfloat16) if args.sym else torch.empty_like(x)
        fn = lambda: hc.allreduce(x, y, comm)
    elif args.op == "rs":
        y = torch.empty(count // world, dtype=x.dtype, device="cuda")
        fn = lambda: hc.reduce_scatter(x, y, comm)
    elif args.op == "ag":
        xs = x[: count // world]
        y = torch.empty(count, dtype=x.dtype, device="cuda")
        fn = lambda: hc.all_gather(xs, y, comm)
    else:
        y = torch.empty_like(x)
        fn = lambda: hc.broadcast(x, y, 0, comm)
    for _ in range(3):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
    fn()
    torch.cuda.synchronize()
    tr = hc.hetccl_comm_get_trace(comm)
    np.save(os.path.join(args.out, f"trace_{args.op}_r{rank}.npy"), tr)
    if rank == 0:
        summarize(tr, f"{args.op} n={world} {args.mib} MiB rank 0 (nch={tr.shape[1]})")
    dist.barrier()
    hc.hetccl_comm_destroy(comm)


if __name__ == "__main__":
    main()
