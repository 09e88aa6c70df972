"""N > 1 host logic on CPU (world_size 2 and 4 over gloo, 127.0.0.1): every rank computes its own plan
from the C ABI and the ranks check, through real collectives, what the one-process-per-GPU path relies
on — identical map validation and active stages on every rank, symmetric signal/wait sets across
processes, conserved per-rank byte counts — plus bench.py's max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, maps, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    import paper_2601_22585_b200 as hc
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for m in maps:
            # 1. map validation and domain count agree on every rank
            nd = hc.hetccl_validate_map(m)
            got = [None] * world
            dist.all_gather_object(got, nd)
            assert len(set(got)) == 1
            for op in range(6):
                plan = hc.hetccl_plan_stages(m, rank, op, root=world - 1)
                plans = [None] * world
                dist.all_gather_object(plans, plan)
                assert len({p["active"] for p in plans}) == 1
                # 2. every signal I send is awaited by its receiver (and nothing else is awaited from me)
                for s in range(plan["nstages"]):
                    c, mask = plan["sig_ctr"][s], plan["sig_mask"][s]
                    for r in range(world):
                        if (mask >> r) & 1:
                            pr = plans[r]
                            assert any(pr["wait_ctr"][s2] == c and (pr["wait_mask"][s2] >> rank) & 1 and s2 > s
                                       for s2 in range(pr["nstages"]))
                for r, pr in enumerate(plans):
                    for s2 in range(pr["nstages"]):
                        if (pr["wait_mask"][s2] >> rank) & 1:
                            assert any(plan["sig_ctr"][s] == pr["wait_ctr"][s2] and (plan["sig_mask"][s] >> r) & 1
                                       for s in range(plan["nstages"]))
                # 3. bytes sent by all ranks == bytes received by all ranks (sum over processes)
                info = hc.hetccl_plan_info(m, rank, op, 1 << 22, hc.BFLOAT16, root=world - 1)
                t = torch.tensor([info["bytes_sent"], info["bytes_recv"]], dtype=torch.int64)
                dist.all_reduce(t)
                assert t[0].item() == t[1].item()
        # 4. bench.py's timing rule: the reported time is the max over ranks
        t = torch.tensor([1.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == float(world)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,maps", [
    (2, [[0, 1], [0, 0]]),
    (4, [[0, 0, 1, 1], [0, 1, 1, 1], [0, 1, 2, 2], [0, 0, 0, 0], [0, 1, 2, 3], [1, 0, 1, 0]]),
])
def test_plan_consistent_across_processes(world, maps):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, maps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
