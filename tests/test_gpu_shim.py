"""NCCL-symbol interposition (§4.4 "zero code modification"): unmodified
torch.distributed code under LD_PRELOAD=libhetccl_nccl.so gets the hierarchical collectives — the
All-Reduce / Reduce-Scatter results are bitwise the oracle's (domain-major order), and the shim reports
the calls it routed to libhetccl.so."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


# one rank runs on a one-GPU box (the shim attaches, every collective is libhetccl's n = 1 copy)
@pytest.mark.parametrize("domains", ["0", pytest.param("0,1", marks=pytest.mark.multigpu),
                                     pytest.param("0,0,1,1", marks=pytest.mark.multigpu)])
def test_ld_preload_shim(domains):
    import torch
    n = len(domains.split(","))
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    shim = os.path.join(ROOT, "paper_2601_22585_b200", "libhetccl_nccl.so")
    assert os.path.exists(shim), "build with __graft_entry__.build()"
    env = dict(os.environ, LD_PRELOAD=shim, HETCCL_DOMAINS=domains, HETCCL_TIMEOUT_S="20")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29711 + n}", os.path.join(ROOT, "tests", "shim_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = next(l for l in out.stdout.splitlines() if l.startswith("SHIM_RESULT "))
    res = json.loads(line[len("SHIM_RESULT "):])
    for r in res:
        assert r["ok"], res
        # 3 all-reduce + reduce-scatter + all-gather went through hetccl (one rank: torch does the all-gather
        # of a single block itself)
        assert r["routed"] >= (5 if n > 1 else 4), res
