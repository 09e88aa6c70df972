"""Drop-in integration with PyTorch DDP (the paper's "zero code modification" goal,
PAPER.md:275-277 §4.4): a DDP communication hook that all-reduces every gradient bucket with the
hierarchical All-Reduce of libhetccl.so instead of NCCL.

    import paper_2601_22585_b200 as hc
    from paper_2601_22585_b200.ddp import HetcclHookState, hetccl_allreduce_hook
    state = HetcclHookState(rank_to_domain=[0, 0, 1, 1])       # after dist.init_process_group
    ddp_model.register_comm_hook(state, hetccl_allreduce_hook)

The bucket is reduced in place (sum, in the oracle's domain-major order) and then divided by the world size,
as DDP's default hook does. The All-Reduce runs on the state's own communication stream, ordered after the
gradient producer by a stream wait and returned as a CUDA-aware future, so DDP's backward keeps computing the
next buckets while this one is on the wire (DDP's finalize makes its stream wait for the future). The comm is
created with `nchannels` CTAs per op (default 64 of the GPU's 296 slots of the legacy kernels) so the backward
kernels keep SMs to run on. Bootstrap uses a gloo group for the IPC blob exchange; the data path never
touches NCCL. For a whole process group on libhetccl see `dist_backend` (backend "hetccl").
"""
import os

import torch
import torch.distributed as dist

from . import BFLOAT16, FLOAT16, FLOAT32, hetccl_allreduce, init_process_group_comm

_CODES = {torch.float32: FLOAT32, torch.bfloat16: BFLOAT16, torch.float16: FLOAT16}


class HetcclHookState:
    """Holds the hetccl communicator of this rank (one per DDP model; it must not be shared with another
    stream's concurrent collectives)."""

    def __init__(self, rank_to_domain, group=None, average=True, nchannels=64, stream=None):
        self.world = dist.get_world_size(group)
        if len(rank_to_domain) != self.world:
            raise ValueError("rank_to_domain must have one entry per rank")
        self.gloo = dist.new_group(backend="gloo")
        old = os.environ.get("HETCCL_NCHANNELS")
        if nchannels:
            os.environ["HETCCL_NCHANNELS"] = str(int(nchannels))
        try:
            self.comm = init_process_group_comm(list(rank_to_domain), group=self.gloo)
        finally:
            if nchannels:
                if old is None:
                    os.environ.pop("HETCCL_NCHANNELS", None)
                else:
                    os.environ["HETCCL_NCHANNELS"] = old
        self.average = average
        self.stream = stream or torch.cuda.Stream()


def hetccl_allreduce_hook(state, bucket):
    buf = bucket.buffer()
    if buf.dtype not in _CODES:
        raise TypeError(f"hetccl hook: unsupported gradient dtype {buf.dtype}")
    main = torch.cuda.current_stream(buf.device)
    state.stream.wait_stream(main)  # the bucket's gradients are complete on the comm stream
    with torch.cuda.stream(state.stream):
        hetccl_allreduce(buf.data_ptr(), buf.data_ptr(), buf.numel(), _CODES[buf.dtype], "sum", state.comm,
                         state.stream.cuda_stream)
        if state.average:
            buf.div_(state.world)
        buf.record_stream(state.stream)
        fut = torch.futures.Future(devices=[buf.device])
        fut.set_result(buf)  # CUDA-aware: waiters' streams wait for this point of the comm stream
    return fut
