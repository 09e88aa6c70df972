"""torch.distributed backend "hetccl" (the paper's "zero code modification" goal, PAPER.md:275-277
§4.4): the collectives of a process group run on libhetccl.so's hierarchical kernels instead of NCCL.

    import torch.distributed as dist
    import paper_2601_22585_b200.dist_backend            # registers the backend
    # HETCCL_DOMAINS="0,0,1,1" gives the rank -> domain map (default: one domain)
    dist.init_process_group("hetccl", rank=r, world_size=n)   # or dist.new_group(backend="hetccl")
    dist.all_reduce(t)            # t a CUDA tensor: hetccl_allreduce on the current stream

A Python ProcessGroup (torch's pybind trampoline) that only marshals arguments into the C ABI: every collective
is one libhetccl call enqueued on the caller's current CUDA stream, so `async_op=False` ordering is the stream
order and a returned Work completes with the stream. Bootstrap: the IPC blobs travel through the process group's
c10d Store (no gloo group needed); ranks agree on success before the group is usable. DDP works on top of it
(its reducer calls ProcessGroup.allreduce). Supported: all_reduce (sum / max / min / avg), broadcast, reduce,
all_gather(_into_tensor), reduce_scatter(_tensor), all_to_all_single with equal splits, barrier; CUDA tensors of
int32 / fp32 / bf16 / fp16. Anything else raises.
"""
import os
import time

import torch
import torch.distributed as dist
from torch._C._distributed_c10d import (AllgatherOptions, AllreduceOptions, AllToAllOptions, BarrierOptions,
                                        BroadcastOptions, ReduceOptions, ReduceScatterOptions,
                                        _create_work_from_future)
from torch.futures import Future

from . import (MAX, MIN, SUM, HetcclError, dtype_code, hetccl_all_gather, hetccl_all_to_all, hetccl_allreduce,
               hetccl_broadcast, hetccl_comm_connect, hetccl_comm_destroy, hetccl_comm_export, hetccl_comm_init,
               hetccl_reduce, hetccl_reduce_scatter)

BACKEND = "hetccl"


def _red(op):
    """(hetccl op, divide-by-world-size?) for a c10d ReduceOp."""
    if op == dist.ReduceOp.SUM:
        return SUM, False
    if op == dist.ReduceOp.AVG:
        return SUM, True
    if op == dist.ReduceOp.MAX:
        return MAX, False
    if op == dist.ReduceOp.MIN:
        return MIN, False
    raise HetcclError(4, f"hetccl backend: unsupported reduce op {op}")


def _domains(size):
    env = os.environ.get("HETCCL_DOMAINS")
    if not env:
        return [0] * size
    m = [int(v) for v in env.split(",")]
    if len(m) != size:
        raise HetcclError(4, f"HETCCL_DOMAINS has {len(m)} entries for a group of {size}")
    return m


def _bits(t):
    """(dtype code, element count) for a pure data movement (all-gather, broadcast, all-to-all): the tensor's
    bytes as 32-bit or 16-bit words whatever its dtype (DDP all-gathers int64 shapes, for instance)."""
    try:
        return dtype_code(t.dtype), t.numel()
    except HetcclError:
        nb = t.numel() * t.element_size()
        if nb % 4 == 0:
            return dtype_code(torch.int32), nb // 4
        if nb % 2 == 0:
            return dtype_code(torch.float16), nb // 2
        raise HetcclError(4, f"hetccl backend: {t.dtype} tensor of {nb} bytes is not a whole number of 16-bit words")


def _cuda(t):
    if not t.is_cuda:
        raise HetcclError(5, "hetccl backend: tensors must be CUDA tensors")
    if not t.is_contiguous():
        raise HetcclError(4, "hetccl backend: tensors must be contiguous")
    return t


class ProcessGroupHetccl(dist.ProcessGroup):
    def __init__(self, store, rank, size, timeout=None, rank_to_domain=None):
        super().__init__(rank, size)
        self._rank, self._size = rank, size
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.rank_to_domain = list(rank_to_domain) if rank_to_domain is not None else _domains(size)
        self.comm = hetccl_comm_init(size, rank, self.rank_to_domain, self.device.index)
        ok = 1
        try:
            store.set(f"hetccl/blob/{rank}", hetccl_comm_export(self.comm))
            blobs = [store.get(f"hetccl/blob/{r}") for r in range(size)]
            hetccl_comm_connect(self.comm, blobs)
        except HetcclError:
            ok = 0
        # agreement: the group is usable only if every rank connected (a rank that failed must not leave the
        # others spinning in their first collective)
        store.add("hetccl/failed", 1 - ok)
        store.add("hetccl/arrived", 1)
        limit = time.monotonic() + (timeout.total_seconds() if timeout is not None else 1800.0)
        while store.add("hetccl/arrived", 0) < size:
            if time.monotonic() > limit:
                raise HetcclError(2, "hetccl backend: timed out waiting for every rank to connect")
            time.sleep(0.001)
        if store.add("hetccl/failed", 0):
            hetccl_comm_destroy(self.comm)
            self.comm = None
            raise HetcclError(2, "hetccl backend: a rank failed to connect its communicator")

    # ---------------------------------------------------------------- plumbing
    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def _done(self, result):
        fut = Future(devices=[self.device])
        fut.set_result(result)
        return _create_work_from_future(fut)

    def size(self):
        return self._size

    def getBackendName(self):
        return BACKEND

    # ---------------------------------------------------------------- collectives
    def allreduce(self, tensors, opts=AllreduceOptions()):
        op, avg = _red(opts.reduceOp)
        for t in tensors:
            _cuda(t)
            hetccl_allreduce(t.data_ptr(), t.data_ptr(), t.numel(), dtype_code(t.dtype), op, self.comm, self._stream())
            if avg:
                t.div_(self._size)
        return self._done(tensors)

    def allreduce_coalesced(self, tensors, opts=AllreduceOptions()):
        return self.allreduce(tensors, opts)

    def broadcast(self, tensors, opts=BroadcastOptions()):
        for t in tensors:
            _cuda(t)
            code, cnt = _bits(t)
            hetccl_broadcast(t.data_ptr(), t.data_ptr(), cnt, code, opts.rootRank, self.comm, self._stream())
        return self._done(tensors)

    def reduce(self, tensors, opts=ReduceOptions()):
        op, avg = _red(opts.reduceOp)
        for t in tensors:
            _cuda(t)
            hetccl_reduce(t.data_ptr(), t.data_ptr(), t.numel(), dtype_code(t.dtype), op, opts.rootRank, self.comm,
                          self._stream())
            if avg and self._rank == opts.rootRank:
                t.div_(self._size)
        return self._done(tensors)

    def _allgather_base(self, output, input, opts=AllgatherOptions()):
        _cuda(output), _cuda(input)
        if output.numel() != input.numel() * self._size:
            raise HetcclError(4, "all_gather: output must hold world_size inputs")
        code, cnt = _bits(input)
        hetccl_all_gather(input.data_ptr(), output.data_ptr(), cnt, code, self.comm, self._stream())
        return self._done(output)

    def allgather_into_tensor_coalesced(self, outputs, inputs, opts=AllgatherOptions()):
        for o, i in zip(outputs, inputs):
            self._allgather_base(o, i, opts)
        return self._done(outputs)

    def allgather(self, output_lists, inputs, opts=AllgatherOptions()):
        for outs, inp in zip(output_lists, inputs):
            flat = torch.empty(inp.numel() * self._size, dtype=inp.dtype, device=inp.device)
            self._allgather_base(flat, _cuda(inp).contiguous(), opts)
            for r, o in enumerate(outs):
                o.copy_(flat[r * inp.numel():(r + 1) * inp.numel()].view_as(o))
        return self._done(output_lists)

    def _reduce_scatter_base(self, output, input, opts=ReduceScatterOptions()):
        op, avg = _red(opts.reduceOp)
        _cuda(output), _cuda(input)
        if input.numel() != output.numel() * self._size:
            raise HetcclError(4, "reduce_scatter: input must hold world_size outputs")
        hetccl_reduce_scatter(input.data_ptr(), output.data_ptr(), output.numel(), dtype_code(output.dtype), op,
                              self.comm, self._stream())
        if avg:
            output.div_(self._size)
        return self._done(output)

    def reduce_scatter_tensor_coalesced(self, outputs, inputs, opts=ReduceScatterOptions()):
        for o, i in zip(outputs, inputs):
            self._reduce_scatter_base(o, i, opts)
        return self._done(outputs)

    def reduce_scatter(self, outputs, input_lists, opts=ReduceScatterOptions()):
        for out, ins in zip(outputs, input_lists):
            flat = torch.cat([i.reshape(-1) for i in ins])
            self._reduce_scatter_base(_cuda(out), flat, opts)
        return self._done(outputs)

    def alltoall_base(self, output, input, output_split_sizes, input_split_sizes, opts=AllToAllOptions()):
        if output_split_sizes or input_split_sizes:
            raise HetcclError(4, "all_to_all_single: only equal splits are supported")
        _cuda(output), _cuda(input)
        code, cnt = _bits(input)
        hetccl_all_to_all(input.data_ptr(), output.data_ptr(), cnt // self._size, code, self.comm, self._stream())
        return self._done(output)

    def barrier(self, opts=BarrierOptions()):
        t = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.allreduce([t])
        torch.cuda.current_stream(self.device).synchronize()
        return self._done(None)

    def shutdown(self):
        if getattr(self, "comm", None) is not None:
            hetccl_comm_destroy(self.comm)
            self.comm = None


def _create(store, rank, size, timeout):
    return ProcessGroupHetccl(store, rank, size, timeout)


if BACKEND not in dist.Backend.backend_list:
    dist.Backend.register_backend(BACKEND, _create, devices=["cuda"])
