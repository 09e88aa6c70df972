"""torch.distributed backend "hetccl" and the DDP comm hook (§4.4).

World size 1 runs on a one-GPU box (the library's n = 1 path: every collective is a copy on the device), so the
driver's GPU run exercises the backend's registration, Store bootstrap, option marshalling and DDP on top of
it. Two ranks (one GPU each) check the results against the CPU oracle bitwise and DDP against NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model():
    import torch
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.GELU(), torch.nn.Linear(512, 64)).cuda()


def _train(ddp, steps=3, seed=100):
    import torch
    opt = torch.optim.SGD(ddp.parameters(), lr=0.05)
    g = torch.Generator(device="cuda").manual_seed(seed)
    for _ in range(steps):
        x = torch.randn(32, 256, device="cuda", generator=g)
        loss = ddp(x).square().mean()
        opt.zero_grad()
        loss.backward()
        opt.step()
    torch.cuda.synchronize()
    return torch.cat([p.detach().flatten().cpu() for p in ddp.parameters()])


def test_backend_world1(tmp_path):
    """One rank: every collective through the backend (the n = 1 copy kernel) and DDP on the hetccl group
    (equal to local training bitwise: the all-reduce of one rank is the identity, AVG divides by 1)."""
    import torch
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP
    import paper_2601_22585_b200.dist_backend as db
    store = dist.FileStore(str(tmp_path / "store"), 1)
    dist.init_process_group(db.BACKEND, store=store, rank=0, world_size=1)
    try:
        assert dist.get_backend() == db.BACKEND
        x = torch.randn(4099, device="cuda").bfloat16()
        y = x.clone()
        dist.all_reduce(y)
        assert torch.equal(y, x)
        dist.all_reduce(y, op=dist.ReduceOp.MAX)
        assert torch.equal(y, x)
        out = torch.empty_like(x)
        dist.all_gather_into_tensor(out, x)
        assert torch.equal(out, x)
        rs = torch.empty_like(x)
        dist.reduce_scatter_tensor(rs, x)
        assert torch.equal(rs, x)
        b = x.clone()
        dist.broadcast(b, src=0)
        assert torch.equal(b, x)
        dist.barrier()
        ddp = DDP(_model(), device_ids=[torch.cuda.current_device()])
        got = _train(ddp)
        ref = _train(_model())
        assert torch.equal(got, ref)
    finally:
        dist.destroy_process_group()


def test_ddp_hook_world1(tmp_path):
    """The DDP comm hook on a one-rank NCCL group (its comm stream + CUDA-aware future): equal to plain local
    training bitwise."""
    import torch
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP
    from paper_2601_22585_b200.ddp import HetcclHookState, hetccl_allreduce_hook
    store = dist.FileStore(str(tmp_path / "store"), 1)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1)
    try:
        ddp = DDP(_model(), device_ids=[torch.cuda.current_device()], bucket_cap_mb=1)
        ddp.register_comm_hook(HetcclHookState(rank_to_domain=[0]), hetccl_allreduce_hook)
        got = _train(ddp)
        ref = _train(_model())
        assert torch.equal(got, ref)
    finally:
        dist.destroy_process_group()


def _two_ranks(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), HETCCL_TIMEOUT_S="20", HETCCL_DOMAINS="0,1")
    import torch
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP
    import paper_2601_22585_b200.dist_backend as db
    import synth
    torch.cuda.set_device(rank)
    dist.init_process_group(db.BACKEND, rank=rank, world_size=world)
    try:
        count = 3 * (1 << 20) + 7
        x = synth.normal(9, rank, count, "bf16")
        t = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
        dist.all_reduce(t)
        R = count // world * world
        rs = torch.empty(R // world, dtype=torch.bfloat16, device="cuda")
        src = torch.from_numpy(x[:R].view(np.int16)).view(torch.bfloat16).cuda()
        dist.reduce_scatter_tensor(rs, src)
        ag = torch.empty(R, dtype=torch.bfloat16, device="cuda")
        dist.all_gather_into_tensor(ag, rs)
        torch.cuda.synchronize()
        ddp = DDP(_model(), device_ids=[rank])
        params = _train(ddp, seed=200 + rank)
        q.put((rank, t.cpu().view(torch.int16).numpy().view(np.uint16), ag.cpu().view(torch.int16).numpy(),
               params.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.multigpu
def test_backend_two_ranks_vs_oracle():
    import torch
    import oracle
    import synth
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_two_ranks, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = {}
    for _ in range(2):
        r, ar, ag, params = q.get(timeout=300)
        out[r] = (ar, ag, params)
    for p in ps:
        p.join(timeout=60)
    count = 3 * (1 << 20) + 7
    xs = [synth.normal(9, r, count, "bf16") for r in range(2)]
    want = oracle.allreduce(xs, [0, 1], "bf16", "sum")
    for r in range(2):
        assert np.array_equal(out[r][0], want), f"rank {r} all_reduce"
    assert np.array_equal(out[0][1], out[1][1])  # AG of RS identical on both ranks (== AR prefix)
    assert np.array_equal(out[0][1].view(np.uint16), want[:out[0][1].size])
    np.testing.assert_array_equal(out[0][2], out[1][2])  # DDP replicas identical
