"""NCCL baseline probe: flat ncclAllReduce / ReduceScatter / AllGather bus bandwidth via
torch.distributed on this box. Run under torchrun; rank 0 prints one JSON line per (op, size).
NCCL is the comparison baseline only; it is never on the hetccl product path."""
import json
import os
import sys

import torch
import torch.distributed as dist


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    sizes = [1 << s for s in range(20, 31, 2)] + [256 << 20]
    tag = os.environ.get("PROBE_TAG", "default")
    for op in ("all_reduce", "reduce_scatter", "all_gather"):
        for nbytes in sorted(set(sizes)):
            n = nbytes // 2
            x = torch.randn(n, device="cuda", dtype=torch.bfloat16)
            out = torch.empty(n // world if op == "reduce_scatter" else n, device="cuda", dtype=torch.bfloat16)
            inp_ag = x[: n // world]
            def run():
                if op == "all_reduce":
                    dist.all_reduce(x)
                elif op == "reduce_scatter":
                    dist.reduce_scatter_tensor(out, x)
                else:
                    dist.all_gather_into_tensor(x, inp_ag)
            for _ in range(3):
                run()
            iters = 20 if nbytes <= (64 << 20) else 5
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier(); torch.cuda.synchronize()
            s.record()
            for _ in range(iters):
                run()
            e.record(); torch.cuda.synchronize()
            ms = torch.tensor([s.elapsed_time(e) / iters], device="cuda")
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            t = ms.item() * 1e-3
            algbw = nbytes / t / 1e9
            fac = 2 * (world - 1) / world if op == "all_reduce" else (world - 1) / world
            if rank == 0:
                print(json.dumps({"tag": tag, "op": op, "n": world, "bytes": nbytes, "ms": round(t * 1e3, 4),
                                  "algbw": round(algbw, 1), "busbw": round(algbw * fac, 1)}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
