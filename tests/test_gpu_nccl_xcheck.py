"""cross-check against an external library on real GPUs — int32 sum All-Reduce bitwise equal
to NCCL's (integer addition is order-free), f32 / bf16 sums within DESIGN.md R7's gate of NCCL's result
(reduction orders differ), All-Gather / Broadcast / All-to-All bitwise equal. Two processes, one GPU each."""
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


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), HETCCL_TIMEOUT_S="20")
    import torch
    import torch.distributed as dist
    import paper_2601_22585_b200 as hc
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    res = {}
    try:
        comm = hc.init_process_group_comm(list(range(world)))
        g = torch.Generator(device="cuda").manual_seed(1234 + rank)
        for count in (1000, 3 * (1 << 20) + 7):  # one-shot and pipeline paths
            xi = torch.randint(-2**31, 2**31 - 1, (count,), dtype=torch.int32, device="cuda", generator=g)
            yi = torch.empty_like(xi)
            hc.allreduce(xi, yi, comm)
            ni = xi.clone()
            dist.all_reduce(ni)
            res[f"int32_{count}"] = bool(torch.equal(yi, ni))
            for dt in (torch.float32, torch.bfloat16):
                xf = torch.randn(count, device="cuda", generator=g).to(dt)
                yf = torch.empty_like(xf)
                hc.allreduce(xf, yf, comm)
                nf = xf.clone()
                dist.all_reduce(nf)
                ref = xf.double()
                absum = xf.double().abs()
                dist.all_reduce(ref)
                dist.all_reduce(absum)
                err = (yf.double() - ref).abs()
                ok = bool((err <= 1e-2 * absum + 1e-30).all()) and float((yf.double() - ref).norm() / ref.norm()) <= 1e-2
                ok = ok and bool(((nf.double() - yf.double()).abs() <= 2e-2 * absum + 1e-30).all())
                res[f"{dt}_{count}"] = ok
        x = torch.randn(4099 * world, device="cuda", generator=g).bfloat16()
        ag = torch.empty(4099 * world * world, dtype=x.dtype, device="cuda")
        hc.all_gather(x, ag, comm)
        nag = torch.empty_like(ag)
        dist.all_gather_into_tensor(nag, x)
        res["all_gather"] = bool(torch.equal(ag.view(torch.int16), nag.view(torch.int16)))
        bc = torch.empty_like(x)
        hc.broadcast(x, bc, 1, comm)
        nbc = x.clone()
        dist.broadcast(nbc, src=1)
        res["broadcast"] = bool(torch.equal(bc.view(torch.int16), nbc.view(torch.int16)))
        a2 = torch.empty_like(x)
        hc.all_to_all(x, a2, comm)
        na2 = torch.empty_like(x)
        dist.all_to_all_single(na2, x)
        res["all_to_all"] = bool(torch.equal(a2.view(torch.int16), na2.view(torch.int16)))
        torch.cuda.synchronize()
        hc.hetccl_comm_get_async_error(comm)
        hc.hetccl_comm_destroy(comm)
        q.put((rank, res))
    except Exception as e:  # pragma: no cover
        q.put((rank, {"error": repr(e)}))
    finally:
        dist.destroy_process_group()


def test_against_nccl():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    for r, res in out.items():
        assert res and all(v is True for v in res.values()), (r, res)
