"""DDP communication hook: two processes, one GPU each, train a small model for a few
steps with the hetccl hook and with plain NCCL DDP from the same initial weights and data; the parameters
must agree within bf16/fp32 reduction-order tolerance and the hetccl run must have used libhetccl.so."""
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _train(rank, world, port, use_hetccl, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), HETCCL_TIMEOUT_S="20")
    import torch
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(512, 1024), torch.nn.GELU(), torch.nn.Linear(1024, 256)).cuda()
        ddp = DDP(model, device_ids=[rank], bucket_cap_mb=1)
        if use_hetccl:
            from paper_2601_22585_b200.ddp import HetcclHookState, hetccl_allreduce_hook
            ddp.register_comm_hook(HetcclHookState(rank_to_domain=list(range(world))), hetccl_allreduce_hook)
        opt = torch.optim.SGD(ddp.parameters(), lr=0.05)
        g = torch.Generator(device="cuda").manual_seed(100 + rank)
        for _ in range(5):
            x = torch.randn(64, 512, device="cuda", generator=g)
            loss = ddp(x).square().mean()
            opt.zero_grad()
            loss.backward()
            opt.step()
        torch.cuda.synchronize()
        flat = torch.cat([p.detach().flatten().cpu() for p in model.parameters()])
        q.put((rank, flat.numpy()))
    finally:
        dist.destroy_process_group()


def _run(use_hetccl):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_train, args=(r, 2, port, use_hetccl, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    return out


def test_ddp_hook_matches_nccl():
    import numpy as np
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    a = _run(True)
    b = _run(False)
    np.testing.assert_array_equal(a[0], a[1])  # replicas stay identical (every rank gets the same sum)
    np.testing.assert_allclose(a[0], b[0], rtol=1e-5, atol=1e-6)
