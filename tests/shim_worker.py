"""Worker for tests/test_gpu_shim.py, launched by torchrun with LD_PRELOAD=libhetccl_nccl.so: plain
torch.distributed code (no hetccl import) whose NCCL collectives the shim routes to libhetccl.so."""
import ctypes
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import oracle
    import synth
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    m = [int(v) for v in os.environ["HETCCL_DOMAINS"].split(",")]
    count = 3 * (1 << 20) + 77
    ok = True
    for it in range(3):
        x = synth.normal(90 + it, rank, count, "bf16")
        t = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
        dist.all_reduce(t)  # ncclAllReduce -> hetccl_allreduce
        xs = [synth.normal(90 + it, r, count, "bf16") for r in range(world)]
        want = oracle.allreduce(xs, m, "bf16", "sum")
        ok &= bool(np.array_equal(t.cpu().view(torch.int16).numpy().view(np.uint16), want))
    # reduce-scatter / all-gather / broadcast through the shim as well
    R = 4096 + 5
    xs = [synth.normal(95, r, world * R, "bf16") for r in range(world)]
    xt = torch.from_numpy(xs[rank].view(np.int16)).view(torch.bfloat16).cuda()
    y = torch.empty(R, dtype=torch.bfloat16, device="cuda")
    dist.reduce_scatter_tensor(y, xt)
    ok &= bool(np.array_equal(y.cpu().view(torch.int16).numpy().view(np.uint16),
                              oracle.reduce_scatter(xs, m, "bf16", "sum")[rank]))
    g = torch.empty(world * R, dtype=torch.bfloat16, device="cuda")
    dist.all_gather_into_tensor(g, y)
    torch.cuda.synchronize()
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2601_22585_b200", "libhetccl_nccl.so"))
    routed, passed = ctypes.c_long(0), ctypes.c_long(0)
    lib.hetccl_shim_stats(ctypes.byref(routed), ctypes.byref(passed))
    res = [None] * world
    dist.all_gather_object(res, {"rank": rank, "ok": ok, "routed": routed.value, "passed": passed.value})
    if rank == 0:
        print("SHIM_RESULT " + json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
