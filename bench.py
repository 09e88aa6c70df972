#!/usr/bin/env python
"""bench.py — hierarchical All-Reduce bus bandwidth on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hetccl|reference] [--mib 256]

One "step" = one hierarchical All-Reduce (intra-domain RS -> cross-domain
exchange -> intra-domain AG, one kernel launch) of a 256 MiB bf16 gradient bucket per rank.
* N = 1: the BASELINE configs[1] target point (4+4 domains, 8 ranks, 256 MiB bf16) with all 8 logical
  ranks multiplexed on one B200 (hetccl_comm_init_mux: same kernel, one cooperative launch); every
  "NVLink" byte is local HBM traffic, so the roofline is HBM.
* N > 1 (torchrun, one process per GPU, NCCL process group for barriers/timing only): real NVLink 5
  ranks, domain split N=2 -> 1+1, N=4 -> 2+2, N=8 -> 4+4; roofline = NVLink.
value = bus GB/s (nccl-tests convention, n = logical ranks: algbw * 2(n-1)/n); inputs (256 MiB per
rank) exceed the 126 MB L2, so no flush is needed between steps. Rank 0 prints one JSON line.
--impl reference times the CPU oracle (oracle/, the tier's reference arm) on a bounded sample.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MAPS = {1: [0, 0, 0, 0, 1, 1, 1, 1], 2: [0, 1], 4: [0, 0, 1, 1], 8: [0, 0, 0, 0, 1, 1, 1, 1]}
SPLIT_NAME = {1: "4+4 (8 ranks multiplexed on 1 GPU)", 2: "1+1", 4: "2+2", 8: "4+4"}
SEED = 2  # SURVEY §8(d) C2 seed
NVLINK_PEAK = 770.0  # GB/s per direction, measured peer copy (B200_PROFILING.md)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def gen_inputs(n_ranks, count, first_rank=0):
    """bf16 N(0,1)*2^-4 per (seed, rank, i) via the synth module (host), one array per rank."""
    import synth
    from concurrent.futures import ThreadPoolExecutor
    out = [None] * n_ranks

    def one(r):
        out[r] = synth.normal(SEED, first_rank + r, count, "bf16")
    with ThreadPoolExecutor(max_workers=min(8, n_ranks)) as ex:
        list(ex.map(one, range(n_ranks)))
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


class NvlinkCounter:
    """NVLink bytes this GPU transmitted / received, summed over its links, from NVML field values read
    before and after the timed region (the hardware counter behind "achieved NVLink GB/s"). Tries the
    byte counters (NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES) and falls back to the data-throughput counters
    (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX, KiB); reports which one it used, or why none worked."""
    FIELDS = ((202, 204, 1, "NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES"),
              (138, 139, 1024, "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX (KiB)"))

    def __init__(self, cuda_device):
        self.err, self.h, self.field = None, None, None
        try:
            import pynvml
            import torch
            self.nv = pynvml
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(cuda_device)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            get = getattr(pynvml, "nvmlDeviceGetHandleByPciBusId_v2", None) or pynvml.nvmlDeviceGetHandleByPciBusId
            self.h = get(bus)
            self.links = []
            for l in range(pynvml.NVML_NVLINK_MAX_LINKS):
                try:
                    if pynvml.nvmlDeviceGetNvLinkState(self.h, l) == pynvml.NVML_FEATURE_ENABLED:
                        self.links.append(l)
                except Exception:
                    pass
            for tx, rx, scale, name in self.FIELDS:
                if self._read(tx, rx, scale) is not None:
                    self.field = (tx, rx, scale, name)
                    break
            if self.field is None:
                self.err = f"no NVLink byte counter readable ({len(self.links)} links up)"
        except Exception as e:  # no NVML / no NVLink: report, do not fail the bench
            self.err = f"{type(e).__name__}: {e}"

    def _read(self, tx, rx, scale):
        try:
            req = [(tx, l) for l in self.links] + [(rx, l) for l in self.links]
            vals = self.nv.nvmlDeviceGetFieldValues(self.h, req)
            if not vals or any(v.nvmlReturn != 0 for v in vals):
                return None
            k = len(self.links)
            return (sum(int(v.value.ullVal) for v in vals[:k]) * scale,
                    sum(int(v.value.ullVal) for v in vals[k:]) * scale)
        except Exception:
            return None

    def sample(self):
        return self._read(*self.field[:3]) if self.field else None

    def delta(self, a, b, seconds, steps):
        if self.field is None or a is None or b is None:
            return {"available": False, "why": self.err or "counter read failed"}
        tx, rx = b[0] - a[0], b[1] - a[1]
        return {"available": True, "counter": self.field[3], "links": len(self.links),
                "tx_bytes_per_step": tx // max(1, steps), "rx_bytes_per_step": rx // max(1, steps),
                "tx_GBps": round(tx / seconds / 1e9, 2), "rx_GBps": round(rx / seconds / 1e9, 2)}


def profiled_traffic(key):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    (profiles/ncu_traffic.json, written by tools/ncu_summary.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)[key]
        return d["traffic_bytes"], d["source"]
    except Exception:
        return None, None


def busbw(nbytes, t_s, n):
    alg = nbytes / t_s / 1e9
    return alg, alg * 2 * (n - 1) / n


def oracle_baseline(xs_host, m, recv_dev_list, budget_s=15.0, total_count=None):
    """cpu_baseline leg: the oracle as it stands on a bounded sample of the workload, timed twice — on one
    host thread and on every host core (oracle.allreduce_threaded: elements split across threads, same
    per-element fold, bit-identical) — and the GPU result on the same sample compared with it bitwise (the
    only place bench.py runs oracle/ besides --impl reference). `value`/`cores` are the all-cores run."""
    import oracle
    import torch
    count = xs_host[0].size
    # ~15 ns per element index for 8 ranks single-threaded: bound the sample to the budget
    total = int(total_count or count)
    sample = int(min(count, max(1 << 16, budget_s / (2e-9 * len(m)))))
    xs = [x[:sample] for x in xs_host]
    t0 = time.perf_counter()
    want = oracle.allreduce(xs, m, "bf16", "sum")
    dt1 = time.perf_counter() - t0
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    want_t = oracle.allreduce_threaded(xs, m, "bf16", "sum", threads=cores)
    dtt = time.perf_counter() - t0
    _, bus1 = busbw(sample * 2, dt1, len(m))
    _, bust = busbw(sample * 2, dtt, len(m))
    ok = bool(np.array_equal(want, want_t)) and all(
        bool(np.array_equal(y[:sample].cpu().view(torch.int16).numpy().view(np.uint16), want)) for y in recv_dev_list)
    return {"value": round(bust, 3), "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": f"first {sample} of {total} elements per rank, all {len(m)} ranks, one All-Reduce "
                      f"({dtt:.2f} s on {cores} host threads, elements split across threads; {dt1:.2f} s on 1); "
                      f"busbw convention as value",
            "single_thread": {"value": round(bus1, 3), "unit": "GB/s", "cores": 1},
            "gpu_bitwise_equal_on_sample": ok}


def bf16_to_f64(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def fp64_gate(got_u16, xs_u16):
    """DESIGN.md R7: normwise ||Y-R||/||R|| <= 1e-2 and |Y_i-R_i| <= 1e-2 * sum_r |x_r[i]| vs the fp64 sum R."""
    F = np.stack([bf16_to_f64(x) for x in xs_u16])
    R, A, g = F.sum(0), np.abs(F).sum(0), bf16_to_f64(got_u16)
    ok = bool(np.all(np.abs(g - R) <= 1e-2 * A + 1e-30))
    nrm = float(np.linalg.norm(R))
    return bool(ok and (nrm == 0.0 or float(np.linalg.norm(g - R)) / nrm <= 1e-2))


def gate_windows(recv_dev_list, window_inputs, starts, W):
    """Full-size check on sampled outputs: every local rank's result on 3 windows passes the R7 gate."""
    import torch
    ok = True
    for st, xs in zip(starts, window_inputs):
        for y in recv_dev_list:
            ok = ok and fp64_gate(y[st:st + W].cpu().view(torch.int16).numpy().view(np.uint16), xs)
    return bool(ok)


# ---------------------------------------------------------------------------------- N = 1 (mux)
def run_mux(args):
    import torch
    import paper_2601_22585_b200 as hc
    dev = 0
    torch.cuda.set_device(dev)
    m = MAPS[1]
    n = len(m)
    count = args.mib * (1 << 20) // 2
    S = count * 2
    xs = gen_inputs(n, count)
    sends = [torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to("cuda") for x in xs]
    recvs = [torch.empty_like(s) for s in sends]
    comm = hc.hetccl_comm_init_mux(n, m, dev)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def step():
        hc.mux_allreduce(sends, recvs, comm, stream=sp)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        t_start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    hc.hetccl_comm_get_async_error(comm)
    total_ms = t_start.elapsed_time(t_end)
    launch_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    t_step = total_ms / args.steps * 1e-3
    alg, bus = busbw(S, t_step, n)
    W = 4096
    starts = [0, count // 2 - W // 2, count - W]
    ok = gate_windows(recvs, [[x[st:st + W] for x in xs] for st in starts], starts, W)
    how = f"R7 gate vs fp64 sum on 3 windows x {W} elements x {n} local ranks (bitwise: cpu_baseline)"

    # e2e: host pinned buffers -> device -> All-Reduce -> host, every step
    hin = [torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).pin_memory() for x in xs]
    hout = [torch.empty_like(h).pin_memory() for h in hin]
    e2e_steps = max(1, min(args.steps, 5))

    def e2e_step():
        for r in range(n):
            sends[r].copy_(hin[r], non_blocking=True)
        step()
        for r in range(n):
            hout[r].copy_(recvs[r], non_blocking=True)
    e2e_step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    b.record(stream)
    torch.cuda.synchronize()
    t_e2e = a.elapsed_time(b) / e2e_steps * 1e-3
    _, e2e_bus = busbw(S, t_e2e, n)

    hbm_peak, peak_src = peaks()
    alg_bytes = 2 * n * S  # every rank's input read once + output written once: the design-free minimum
    traffic, tsrc = profiled_traffic(f"mux_ar_{m}_{args.mib}MiB_bf16")
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    cpu = oracle_baseline(xs, m, recvs) if not args.no_cpu_baseline else None
    out = {
        "metric": "allreduce_busbw", "value": round(bus, 2), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded bf16 N(0,1)*2^-4)",
        "config": {"workload": f"C2 target point: hierarchical All-Reduce, {args.mib} MiB bf16 per rank, "
                               f"{SPLIT_NAME[1]}", "ranks": n, "rank_to_domain": m, "count": count,
                   "l2": "inputs > L2 (no flush)", "parallelism": "rank-multiplexed"},
        "algbw": round(alg, 2), "gpu_launches": args.steps,
        "e2e": {"value": round(e2e_bus, 2), "unit": "GB/s", "h2d_bytes_per_step": n * S, "d2h_bytes_per_step": n * S},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                     "note": f"algorithmic = 2*n*S = {alg_bytes} B per launch (each rank's input read + output "
                             f"written once); peak {peak_src}; kernel k_allreduce avg launch {launch_ms:.4f} ms; "
                             f"traffic = dram read+write per launch from {tsrc}"},
        "parity": {"ok": ok, "how": how},
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    hc.hetccl_comm_destroy(comm)
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------------- N > 1
def run_dist(args):
    import torch
    import torch.distributed as dist
    import paper_2601_22585_b200 as hc
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if world not in MAPS:
        raise SystemExit(f"--gpus {world}: no domain split defined (use 2, 4 or 8)")
    m = MAPS[world]
    count = args.mib * (1 << 20) // 2
    S = count * 2
    x = gen_inputs(1, count, first_rank=rank)[0]
    send_plain = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to("cuda")
    comm = hc.init_process_group_comm(m)
    # the gradient bucket and its output live in symmetric buffers (hetccl_mem_*: same offset on every
    # rank): domain peers read x directly (pull) and final pieces go straight into the peers' buffers;
    # plain torch buffers take the staged path (reported beside it)
    send = hc.symmetric_empty(comm, count, torch.bfloat16)
    send.copy_(send_plain)
    recv = hc.symmetric_empty(comm, count, torch.bfloat16)
    recv_staged = torch.empty_like(send)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def step():
        hc.allreduce(send, recv, comm, stream=sp)

    def timed(fn, steps):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        a.record(stream)
        for i in range(steps):
            ev[i][0].record(stream)
            fn()
            ev[i][1].record(stream)
        b.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        tot = torch.tensor([a.elapsed_time(b)], device="cuda")
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        lm = torch.tensor([statistics.mean(p.elapsed_time(q) for p, q in ev)], device="cuda")
        dist.all_reduce(lm, op=dist.ReduceOp.MAX)
        return tot.item(), lm.item()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    nvc = NvlinkCounter(local)
    with ClockSampler(local) as clk:
        c0 = nvc.sample()
        total_ms, launch_ms = timed(step, args.steps)
        c1 = nvc.sample()
    nvl = nvc.delta(c0, c1, total_ms * 1e-3, args.steps)
    # busiest rank's measured NVLink transmit bytes per launch (max over ranks)
    txm = torch.tensor([float(nvl.get("tx_bytes_per_step", -1))], device="cuda")
    dist.all_reduce(txm, op=dist.ReduceOp.MAX)
    nvl["tx_bytes_per_step_max_over_ranks"] = int(txm.item())
    # staged path (plain torch recv buffer) for comparison
    for _ in range(args.warmup):
        hc.allreduce(send_plain, recv_staged, comm, stream=sp)
    staged_ms, _ = timed(lambda: hc.allreduce(send_plain, recv_staged, comm, stream=sp), args.steps)
    _, staged_bus = busbw(S, staged_ms / args.steps * 1e-3, world)
    hc.hetccl_comm_get_async_error(comm)
    t_step = total_ms / args.steps * 1e-3
    alg, bus = busbw(S, t_step, world)

    # full-size check on sampled windows: every rank's inputs are regenerated from the generator
    import synth
    W = 4096
    starts = [0, count // 2 - W // 2, count - W]
    ok = gate_windows([recv], [[synth.normal(SEED, r, W, "bf16", start=st) for r in range(world)] for st in starts],
                      starts, W)
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)

    # NCCL flat all-reduce on the same-size buffer (comparison baseline only): on a plain buffer (matched with
    # our staged path) and on a buffer NCCL registered itself (torch.cuda.MemPool on NCCL's allocator +
    # register_mem_pool: window registration, matched with our symmetric-buffer path)
    nbuf = send.clone()
    for _ in range(args.warmup):
        dist.all_reduce(nbuf)
    nccl_ms, _ = timed(lambda: dist.all_reduce(nbuf), args.steps)
    _, nccl_bus = busbw(S, nccl_ms / args.steps * 1e-3, world)
    nccl_reg = {}
    try:
        backend = dist.group.WORLD._get_backend(torch.device("cuda", local))
        pool = torch.cuda.MemPool(backend.mem_allocator)
        with torch.cuda.use_mem_pool(pool):
            rbuf = torch.empty_like(send)
        backend.register_mem_pool(pool)
        rbuf.copy_(send)
        for _ in range(args.warmup):
            dist.all_reduce(rbuf)
        reg_ms, _ = timed(lambda: dist.all_reduce(rbuf), args.steps)
        _, reg_bus = busbw(S, reg_ms / args.steps * 1e-3, world)
        nccl_reg = {"busbw": round(reg_bus, 2)}
        backend.deregister_mem_pool(pool)
        del rbuf
    except Exception as e:  # registration unavailable: say why, keep the plain comparison
        nccl_reg = {"unavailable": f"{type(e).__name__}: {e}"[:200]}

    # e2e through the public API with pinned host buffers
    hin = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).pin_memory()
    hout = torch.empty_like(hin).pin_memory()

    def e2e_step():
        send.copy_(hin, non_blocking=True)
        step()
        hout.copy_(recv, non_blocking=True)
    e2e_step()
    e2e_steps = max(1, min(args.steps, 5))
    e2e_ms, _ = timed(e2e_step, e2e_steps)
    _, e2e_bus = busbw(S, e2e_ms / e2e_steps * 1e-3, world)

    busiest = max(hc.hetccl_plan_info(m, r, hc.OP_ALLREDUCE, count, hc.BFLOAT16)["bytes_sent"] for r in range(world))
    achieved = busiest / (launch_ms * 1e-3) / 1e9
    clocks = clk.summary()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        # the oracle on a bounded sample: every rank's first elements regenerated from the generator; checked
        # bitwise against this rank's GPU result on the same elements
        ns = min(count, 1 << 22)
        cpu = oracle_baseline([synth.normal(SEED, r, ns, "bf16") for r in range(world)], m, [recv[:ns]],
                              total_count=count)
    dist.barrier()
    hc.hetccl_comm_destroy(comm)
    if rank == 0:
        out = {
            "metric": "allreduce_busbw", "value": round(bus, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded bf16 N(0,1)*2^-4)",
            "config": {"workload": f"hierarchical All-Reduce, {args.mib} MiB bf16 per rank, {SPLIT_NAME[world]}",
                       "ranks": world, "rank_to_domain": m, "count": count, "l2": "inputs > L2 (no flush)",
                       "parallelism": f"dp{world}"},
            "algbw": round(alg, 2), "gpu_launches": args.steps * world,
            "nccl_flat": {"busbw": round(nccl_bus, 2), "ratio": round(bus / nccl_bus, 4),
                          "registered": nccl_reg,
                          "matched": {"symmetric_vs_registered": round(bus / nccl_reg["busbw"], 4)
                                      if "busbw" in nccl_reg else None,
                                      "staged_vs_plain": round(staged_bus / nccl_bus, 4)},
                          "note": "ratio = value (our symmetric buffers) / NCCL on a plain buffer; matched pairs: "
                                  "ours on symmetric buffers vs NCCL on its own registered buffer, ours on plain "
                                  "torch buffers vs NCCL on a plain buffer"},
            "staged_recv": {"busbw": round(staged_bus, 2),
                            "note": "send/recv in plain torch buffers: staged through scratch (value: symmetric buffers)"},
            "e2e": {"value": round(e2e_bus, 2), "unit": "GB/s", "h2d_bytes_per_step": world * S,
                    "d2h_bytes_per_step": world * S},
            "roofline": {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_PEAK, "unit": "GB/s",
                         "frac": round(achieved / NVLINK_PEAK, 4),
                         "traffic": nvl.get("tx_bytes_per_step_max_over_ranks") if nvl.get("available") else None,
                         "note": f"algorithmic = busiest rank's NVLink bytes sent per launch ({busiest} B, plan) / "
                                 f"avg k_allreduce launch {launch_ms:.4f} ms; peak = measured peer copy per direction; "
                                 f"traffic = NVLink bytes transmitted per launch, max over ranks (NVML counter, "
                                 f"this run; an ncu DRAM capture cannot wrap a multi-rank command)"},
            "nvlink_counters": nvl,
            "parity": {"ok": bool(okt.item()), "how": "R7 gate vs fp64 sum on 3 windows x 4096 elements, all ranks"},
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


# ---------------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The tier's reference arm: the CPU oracle as it stands, on the box's host cores (elements split across
    threads by oracle.allreduce_threaded, bit-identical to the serial oracle; the single-thread time is reported
    beside it), each step a bounded sample of the same workload. Rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    import oracle
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    n_gpu = world if world > 1 else args.gpus
    m = MAPS.get(n_gpu, MAPS[1])
    n = len(m)
    count = args.mib * (1 << 20) // 2
    cores = os.cpu_count() or 1
    budget = 150.0  # seconds for warmup + steps together
    per_step = budget / max(1, args.steps + args.warmup)
    sample = int(min(count, max(1 << 14, per_step / (5e-9 * n / min(cores, 8)))))
    xs = gen_inputs(n, sample)
    for _ in range(args.warmup):
        oracle.allreduce_threaded(xs, m, "bf16", "sum", threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.allreduce_threaded(xs, m, "bf16", "sum", threads=cores)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    ns = min(sample, 1 << 22)
    t0 = time.perf_counter()
    oracle.allreduce([x[:ns] for x in xs], m, "bf16", "sum")
    t1 = time.perf_counter() - t0
    _, bus = busbw(sample * 2, t, n)
    _, bus1 = busbw(ns * 2, t1, n)
    workload = (f"C2 target point: hierarchical All-Reduce, {args.mib} MiB bf16 per rank, {SPLIT_NAME[1]}" if n_gpu == 1
                else f"hierarchical All-Reduce, {args.mib} MiB bf16 per rank, {SPLIT_NAME.get(n_gpu, '')}")
    desc = (f"first {sample} of {count} elements per rank, {n} ranks ({SPLIT_NAME.get(n_gpu, '')}), {cores} host threads "
            f"(elements split across threads); single thread on the first {ns}: {bus1:.4f} GB/s")
    out = {
        "impl": "reference", "metric": "allreduce_busbw", "value": round(bus, 4), "unit": "GB/s", "n_gpus": n_gpu,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded bf16 N(0,1)*2^-4)",
        "config": {"workload": workload, "ranks": n, "rank_to_domain": m, "count": count},
        "cpu_baseline": {"value": round(bus, 4), "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": desc,
                         "single_thread": {"value": round(bus1, 4), "unit": "GB/s", "cores": 1}},
        "e2e": {"value": round(bus, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hetccl", choices=["hetccl", "reference"])
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world == 1:
        run_mux(args)
    else:
        run_dist(args)


if __name__ == "__main__":
    main()
