#!/usr/bin/env python
"""Bench: one decode-step attention layer over the hybrid cache (Apt-Serve's hot path).

Metric (BASELINE.json): decode-attention req-layers/s (+ HBM GB/s and tensor-core
utilisation vs the roofline).  One step = one hc_decode_attention call over one batch:
K/V reconstruction of hidden-mode requests (tcgen05 GEMM), split-K attention over KV and
rebuilt K/V, split combine.  Default workload: cfg4 = OPT-66B layer shape, 256 requests,
long contexts (lognormal, <= 4096), 50% hidden, bf16, on one B200.

  python bench.py [--gpus N --steps K --warmup W] [--config cfg4|cfg2|cfg3|cfg5:<h>]
  python bench.py --impl reference ...   # the fp64 CPU oracle as the reference arm

Multi-GPU (one process per GPU; `--gpus N` without torchrun spawns the N ranks itself):
cfg3/cfg4 run STRONG scaling by default — one batch of the recipe split across ranks by LPT on
the cost model, each rank owning its requests' blocks and a W_KV replica —
and every step ends with the NCCL all-gather of every rank's (out, lse) (north_star's output
gather; `--no-gather` drops it).  `--weak` gives every rank its own full batch instead.  The
time is the max over ranks.  The GPU arm never imports oracle/ or tests/: the oracle runs
only in the cpu_baseline leg and in `--impl reference`.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def workload_from(name: str):
    from synth import configs as C
    return C.by_name(name)


def algorithmic(w):
    """bytes and FLOPs the method must move / compute (bf16: s = 2).  dk = Hk*dh
    is the K (or V) row width: d for multi-head, smaller under GQA (R18)."""
    d, s, dk = w.shape.d, w.elem_bytes, w.shape.dk
    kv_tok = w.n_tokens(0)
    hid_tok = w.n_tokens(1)
    n_req = len(w.n)
    bytes_ = kv_tok * 2 * dk * s + hid_tok * d * s + (2 * dk * d * s + 2 * dk * 4 if hid_tok else 0) + 2 * n_req * d * s
    flops = 4 * d * dk * hid_tok
    return bytes_, flops, kv_tok, hid_tok


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t_end = time.time() + 3.0   # nvidia-smi start-up: wait for its first sample
            while not self.lines and time.time() < t_end:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self):
        """Start of the timed region: samples from nvidia-smi's start-up (its first NVML
        queries can stall CUDA calls) and from warm-up are dropped; the sampler is started
        before warm-up so that start-up never lands inside the timed region."""
        self.t0 = time.time()

    def stop(self):
        if self.proc is None:
            return None
        t1 = time.time()
        time.sleep(0.12)   # one more sample period, for timed regions shorter than 100 ms
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sms, smax, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0 = getattr(self, "t0", 0.0)
        window = "timed region"
        lines = [(ts, ln) for ts, ln in self.lines if t0 <= ts <= t1 + 0.01]
        if not lines:   # timed region shorter than the 100 ms sample period
            lines = [(ts, ln) for ts, ln in self.lines if t0 - 0.15 <= ts <= t1 + 0.15]
            window = "timed region +-150 ms (region shorter than the 100 ms sample period)"
        for ts, ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            try:
                pw.append(float(f[3]))
            except ValueError:
                pass
            for nm, val in zip(names, f[5:9]):
                if val.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        if not sms:
            return None
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sms), "power_w": statistics.median(pw) if pw else None, "window": window}


# ============================================================================ reference arm
def run_reference(args, rank: int, world: int):
    if rank != 0:
        return 0
    import numpy as np
    import torch
    from threadpoolctl import threadpool_info

    from oracle import hc_oracle as O
    from synth.configs import MODE_HIDDEN, MODE_KV

    w = workload_from(args.config)
    d, H = w.shape.d, w.shape.H
    rs = np.random.default_rng(1234)
    kv = [i for i in range(len(w.n)) if w.modes[i] == MODE_KV]
    hid = [i for i in range(len(w.n)) if w.modes[i] == MODE_HIDDEN]
    W = None
    if hid:
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        W = w.w_kv(device=dev).cpu()   # synth is bit-identical on any device (tests/test_gpu_parity.py::test_synth_bit_identical_on_device)
    picks = []
    for s in range(args.warmup + args.steps):
        step = []
        if kv:
            step.append(int(rs.choice(kv)))
        if hid:
            step.append(int(rs.choice(hid)))
        picks.append(step)
    Wd = O._f64(W) if W is not None else None
    t_total, n_done = 0.0, 0
    for s, step in enumerate(picks):
        reqs = []
        for i in step:
            r = {"q": w.q(i), "mode": w.modes[i]}
            if w.modes[i] == MODE_KV:
                r["K"], r["V"] = w.kv(i)
            else:
                r["X"] = w.x(i)
            reqs.append(r)
        t0 = time.perf_counter()
        O.decode_batch(reqs, Wd, H, w.scale, w.b_kv(), n_kv_heads=w.shape.n_kv)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            t_total += dt
            n_done += len(step)
    cores = max([tp.get("num_threads", 1) for tp in threadpool_info()] + [1])
    value = n_done / t_total if t_total > 0 else 0.0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "req-layers/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "shape": w.shape.name, "n_req": len(w.n), "note": w.note},
        "cpu_baseline": {"value": value, "unit": "req-layers/s", "cores": cores, "kind": "oracle",
                         "sample": f"per step 1 KV + 1 hidden request of {w.name} drawn with seed 1234 "
                                   f"(full heads, fp64 numpy oracle)"},
        "e2e": {"value": value, "unit": "req-layers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "decode-attention req-layers/s (hybrid KV/hidden cache, one layer)"


# ============================================================================ CPU baseline
def cpu_baseline(w, budget_s: float = 20.0):
    """The oracle as it stands, on a bounded sample of the same workload (rank 0, N=1)."""
    import numpy as np
    import torch
    from threadpoolctl import threadpool_info

    from oracle import hc_oracle as O
    from synth.configs import MODE_HIDDEN, MODE_KV

    H = w.shape.H
    rs = np.random.default_rng(99)
    kv = [i for i in range(len(w.n)) if w.modes[i] == MODE_KV]
    hid = [i for i in range(len(w.n)) if w.modes[i] == MODE_HIDDEN]
    Wd = O._f64(w.w_kv(device="cuda").cpu()) if hid else None
    b = w.b_kv()
    order = []
    # alternate KV / hidden picks in the workload's proportion until the budget is spent
    pool_kv, pool_h = list(rs.permutation(kv)) if kv else [], list(rs.permutation(hid)) if hid else []
    t_used, n_kv, n_h = 0.0, 0, 0
    t_kv, t_h = 0.0, 0.0
    while t_used < budget_s and (pool_kv or pool_h):
        for src, is_h in ((pool_kv, False), (pool_h, True)):
            if not src or t_used >= budget_s:
                continue
            i = int(src.pop())
            r = {"q": w.q(i), "mode": w.modes[i]}
            if is_h:
                r["X"] = w.x(i)
            else:
                r["K"], r["V"] = w.kv(i)
            t0 = time.perf_counter()
            O.decode_batch([r], Wd, H, w.scale, b, n_kv_heads=w.shape.n_kv)
            dt = time.perf_counter() - t0
            t_used += dt
            if is_h:
                n_h, t_h = n_h + 1, t_h + dt
            else:
                n_kv, t_kv = n_kv + 1, t_kv + dt
            order.append(i)
    # whole-batch extrapolation in the workload's own mix: per-request mean times
    frac_h = len(hid) / len(w.n)
    per_req = (1 - frac_h) * (t_kv / max(1, n_kv)) + frac_h * (t_h / max(1, n_h))
    cores = max([tp.get("num_threads", 1) for tp in threadpool_info()] + [1])
    # one thread, for reference: the shortest KV and hidden requests, per token
    single = {}
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            for key, src in (("kv_token_us", kv), ("hidden_token_us", hid)):
                if not src:
                    continue
                i = min(src, key=lambda j: w.n[j])
                r = {"q": w.q(i), "mode": w.modes[i]}
                if w.modes[i] == MODE_HIDDEN:
                    r["X"] = w.x(i)
                else:
                    r["K"], r["V"] = w.kv(i)
                t0 = time.perf_counter()
                O.decode_batch([r], Wd, H, w.scale, b, n_kv_heads=w.shape.n_kv)
                single[key] = (time.perf_counter() - t0) / w.n[i] * 1e6
    except Exception as ex:   # reported, not fatal: the multi-thread number is the baseline
        single = {"error": f"{type(ex).__name__}: {ex}"[:200]}
    return {"value": 1.0 / per_req if per_req > 0 else 0.0, "unit": "req-layers/s", "cores": cores,
            "single_thread": single,
            "kind": "oracle", "extrapolated": True,
            "kv_req_layers_per_s": n_kv / t_kv if t_kv > 0 else None,
            "hidden_req_layers_per_s": n_h / t_h if t_h > 0 else None,
            "sample": f"{n_kv} KV + {n_h} hidden requests of {w.name} (seed 99, full heads, fp64 numpy), "
                      f"{t_used:.1f} s; value = 1 / (mix-weighted mean time per request)"}


# ============================================================================ phase-2 strong scaling
def run_split(args, rank: int, world: int, local: int, w0):
    """Strong scaling with token-range splitting (SURVEY §8(e) phase 2): every rank holds
    its parts of the batch (synth.partition.lpt_split), decodes them, all-gathers (out,
    lse) and merges every request's parts with hc_merge_partials.  All of it is timed."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2504_07494_b200 import hc
    from synth.configs import MODE_KV
    from synth import drive as T
    from synth.partition import lpt_split

    d, Hh, B = w0.shape.d, w0.shape.H, w0.block_size
    plans = lpt_split(w0.n, w0.modes, d, world, B)
    mine = plans[rank]
    wr = w0.subset(sorted({i for i, _, _ in mine}) or [0])
    dt = hc.HC_BF16 if w0.dtype == "bf16" else hc.HC_F32
    nblk = sum(hc.units_needed(d, Hh, w0.shape.dh, B, w0.modes[i], t1 - t0, dt) for i, t0, t1 in mine)
    pool = T.make_pool(wr, device=local, num_blocks=int(nblk * 1.05) + 8)
    dev = torch.device("cuda", local)
    pid = [10_000_000 + 100_000 * rank + j for j in range(len(mine))]
    for j, (i, t0, t1) in enumerate(mine):   # one part at a time (cache fill, untimed)
        if w0.modes[i] == MODE_KV:
            k, v = w0.kv(i, device=dev, rows=(t0, t1))
            pool.append([pid[j]], [MODE_KV], [t1 - t0], k=k.contiguous(), v=v.contiguous())
        else:
            pool.append([pid[j]], [1], [t1 - t0], x=w0.x(i, device=dev, rows=(t0, t1)).contiguous())
    q = torch.stack([w0.q(i, device=dev) for i, _, _ in mine]).contiguous() if mine else None
    n_mine = len(mine)
    out_p = torch.empty((max(n_mine, 1), d), dtype=w0.torch_dtype, device=dev)
    lse_p = torch.empty((max(n_mine, 1), Hh), dtype=torch.float32, device=dev)
    ws = pool.workspace(pid) if mine else None
    n_max = max(len(p) for p in plans)
    send = torch.zeros((n_max, d + Hh), dtype=torch.float32, device=dev)
    send[:, d:] = float("-inf")
    recv = torch.empty((world * n_max + 1, d + Hh), dtype=torch.float32, device=dev)
    recv[-1, :d] = 0.0
    recv[-1, d:] = float("-inf")   # the "empty part" row
    # merge index: part p of request i lives in recv row rank * n_max + slot
    parts_of = [[] for _ in w0.n]
    for r, items in enumerate(plans):
        for j, (i, _, _) in enumerate(items):
            parts_of[i].append(r * n_max + j)
    P = max(len(x) for x in parts_of)
    idx = torch.full((P, len(w0.n)), world * n_max, dtype=torch.int64)
    for i, rows in enumerate(parts_of):
        for p, row in enumerate(rows):
            idx[p, i] = row
    idx = idx.to(dev)
    out_all = torch.empty((len(w0.n), d), dtype=torch.float32, device=dev)
    lse_all = torch.empty((len(w0.n), Hh), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        if mine:
            hc.hc_decode_attention(pool.handle, pid, q, w0.scale, out_p, lse_p, ws, stream)
            send[:n_mine, :d].copy_(out_p[:n_mine])
            send[:n_mine, d:].copy_(lse_p[:n_mine])
        if world > 1:
            dist.all_gather_into_tensor(recv[:world * n_max], send)
        else:
            recv[:n_max].copy_(send)
        outs = recv[:, :d].index_select(0, idx.view(-1)).view(P, len(w0.n), d)
        lses = recv[:, d:].index_select(0, idx.view(-1)).view(P, len(w0.n), Hh)
        hc.hc_merge_partials(outs, lses, out_all, lse_all, stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    n_split = sum(1 for x in parts_of if len(x) > 1)
    dump = os.environ.get("HC_BENCH_DUMP")
    if rank == 0 and dump:
        # test hook: the merged (out, lse) of every request, checked against the oracle by
        # tests/test_multiproc.py (the bench itself never runs the oracle on this path)
        np.savez(dump, out=out_all.cpu().numpy(), lse=lse_all.cpu().numpy(),
                 parts=np.array([len(x) for x in parts_of]))
    if rank == 0:
        print(json.dumps({
            "metric": "decode-attention req-layers/s (hybrid KV/hidden cache, one layer)",
            "value": len(w0.n) / (ms / 1e3), "unit": "req-layers/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": w0.dtype, "data": "synthetic",
            "config": {"workload": w0.name, "parallelism": f"request-sharded x{world} (strong, LPT + token-range split)",
                       "split_requests": n_split, "max_parts": P,
                       "output": "all-gather of (out, lse) parts + hc_merge_partials, every step (timed)"},
            "gpu_launches": (pool.last_launch_count() + 1) * args.steps}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ============================================================================ launch plumbing
def spawn_ranks(n: int, build: bool = True) -> int:
    """`python bench.py --gpus N` outside torchrun: build libhc.so once, then launch N ranks
    (one process per GPU) through torch.distributed.run on 127.0.0.1 with the same arguments;
    rank 0's JSON line is this process's output."""
    import socket
    if build:
        from paper_2504_07494_b200 import build as hb
        hb.build()
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def init_dist(local: int):
    """One process group per job: NCCL over NVLink (device-bound) — HC_BENCH_BACKEND=gloo is
    the CPU test hook.  NCCL's INIT log stays on (stderr) so the communicator's rank count is
    on record."""
    import torch
    import torch.distributed as dist
    backend = os.environ.get("HC_BENCH_BACKEND", "nccl")
    if backend == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)


def shard_workload(args, w0, rank: int, world: int):
    """This rank's requests: LPT share of one batch (strong) or its own full batch (weak)."""
    from synth import configs as C
    if args.strong:
        from synth.partition import strong_shard
        return strong_shard(w0, rank, world)
    return C.shard_for_rank(w0, rank, world)


def max_over_ranks(x: float, world: int, device) -> float:
    """Every multi-GPU time is the max over ranks (all-reduce MAX of the device-timed value)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class OutputGather:
    """north_star's output gather: every step, each rank's (out, lse) rows (padded to the
    largest shard) are all-gathered so every rank holds the whole batch's output."""

    def __init__(self, w, n_req: int, world: int, device):
        import torch
        import torch.distributed as dist
        n_max = torch.tensor([n_req], device=device)
        dist.all_reduce(n_max, op=dist.ReduceOp.MAX)
        self.n_req, self.n_max, self.d, self.H = n_req, int(n_max.item()), w.shape.d, w.shape.H
        self.send = torch.zeros((self.n_max, self.d + self.H), dtype=torch.float32, device=device)
        self.recv = torch.empty((world * self.n_max, self.d + self.H), dtype=torch.float32, device=device)

    def __call__(self, out, lse):
        import torch.distributed as dist
        self.send[:self.n_req, :self.d].copy_(out)
        self.send[:self.n_req, self.d:].copy_(lse)
        dist.all_gather_into_tensor(self.recv, self.send)

    def describe(self) -> str:
        import torch.distributed as dist
        return (f"{dist.get_backend()} all-gather of out+lse every step (timed), "
                f"{self.recv.numel() * 4} B gathered per step")


def run_dry(args, rank: int, world: int) -> int:
    """Test hook (HC_BENCH_DRY=1, CPU, gloo): the N>1 control path of the main arm — rank
    plumbing, strong/weak sharding, the output gather, barriers and the max over ranks — with
    zero-filled outputs in place of the decode kernel, timed on the host clock.  Prints the
    same line shape with "dry": true; never a bench number."""
    import torch
    import torch.distributed as dist
    if world > 1:
        init_dist(0)
    w0 = workload_from(args.config)
    args.strong = strong_default(args, w0, world)
    w = shard_workload(args, w0, rank, world)
    n_req = len(w.n)
    out = torch.zeros((n_req, w.shape.d))
    lse = torch.zeros((n_req, w.shape.H))
    gather = OutputGather(w, n_req, world, "cpu") if (not args.no_gather and world > 1) else None
    for _ in range(args.warmup):
        if gather:
            gather(out, lse)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if gather:
            gather(out, lse)
    if world > 1:
        dist.barrier()
    ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / max(args.steps, 1), world, "cpu")
    n_total = len(w0.n) if args.strong else world * n_req
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": n_total / (ms / 1e3), "unit": "req-layers/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "dry": True,
                          "scaling": "strong" if args.strong else "weak",
                          "config": {"workload": w.name, "n_req_per_rank0": n_req, "n_req_total": n_total,
                                     "output_gather": gather.describe() if gather else "none"}}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def strong_default(args, w0, world: int) -> bool:
    """cfg3/cfg4 (and the cfg5 sweep) are strong-scaling configurations — a
    fixed batch split across ranks; cfg2 and `--weak` keep a full batch per rank."""
    if args.weak or world == 1:
        return False
    return args.strong or args.split or w0.name.split("-")[0] in ("cfg3", "cfg4", "cfg5")


# ============================================================================ main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hc", choices=["hc", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--split-tokens", type=int, default=0)
    ap.add_argument("--mode", default="decode", choices=["decode", "layer", "prefill"],
                    help="decode: the north-star hot path (default); layer: hc_decode_layer (q/k/v "
                         "projection + cache write, attention, W_O); prefill: hc_prefill_layer")
    ap.add_argument("--prefill-len", type=int, default=1024)
    ap.add_argument("--prefill-reqs", type=int, default=16)
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: one batch split across ranks by LPT (default for cfg3/cfg4/cfg5)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank processes its own full batch of the recipe")
    ap.add_argument("--rope", type=float, default=0.0,
                    help="RoPE base theta (NEXT row f4 (i)): rebuilt K rotated at its positions")
    ap.add_argument("--absorb", action="store_true",
                    help="NON-PAPER variant (NEXT row f4 (ii)): hidden requests attend through "
                         "q~ = W_K^T q and W_V (sum a x) instead of rebuilding K/V")
    ap.add_argument("--split", action="store_true",
                    help="with --strong: split requests costlier than total/world across ranks "
                         "(SURVEY §8(e) phase 2) and merge their (out, lse) parts after an all-gather")
    ap.add_argument("--no-gather", action="store_true",
                    help="N>1: skip the all-gather of every rank's out + lse over NCCL after each step "
                         "(north_star's output gather, on by default, inside the timed region)")
    ap.add_argument("--fill", default="rr", choices=["rr", "seq"],
                    help="cache fill order: rr = one block per request per round (blocks strided across the "
                         "pool, the default recipe); seq = request by request (consecutive block ids)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay variant")
    ap.add_argument("--profile-steps", type=int, default=0,
                    help="run only N untimed steps (for ncu); prints nothing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.profile_steps == 0 else args.warmup
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus, build=not os.environ.get("HC_BENCH_DRY"))

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("HC_BENCH_ONE_GPU"):
        # test hook: every rank on device 0 (exercises the N>1 control path on a 1-GPU box;
        # use with HC_BENCH_BACKEND=gloo — NCCL refuses two ranks on one GPU)
        local = 0
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if os.environ.get("HC_BENCH_DRY"):
        return run_dry(args, rank, world)
    if args.mode != "decode":
        return run_module_mode(args, rank, world, local)

    import torch
    import torch.distributed as dist

    from paper_2504_07494_b200 import build as hb
    hb.build()   # file-locked: concurrent ranks wait for one build
    from paper_2504_07494_b200 import hc
    from synth import configs as C
    from synth import drive as T

    torch.cuda.set_device(local)
    if world > 1:
        init_dist(local)
    w0 = workload_from(args.config)
    args.strong = strong_default(args, w0, world)
    if args.split:
        return run_split(args, rank, world, local, w0)
    w = shard_workload(args, w0, rank, world)
    pool = T.make_pool(w, device=local, split_tokens=args.split_tokens,
                       flags=hc.HC_FLAG_ABSORB_HIDDEN if args.absorb else 0, rope_theta=args.rope)
    T.fill(pool, w, device=local, order=args.fill)
    q = T.queries(w, device=local)
    ids = list(w.req_ids)
    n_req = len(ids)
    out = torch.empty((n_req, w.shape.d), dtype=w.torch_dtype, device="cuda")
    lse = torch.empty((n_req, w.shape.H), dtype=torch.float32, device="cuda")
    ws = pool.workspace(ids)
    stream = torch.cuda.current_stream()

    gather = OutputGather(w, n_req, world, "cuda") if (not args.no_gather and world > 1) else None

    def step():
        hc.hc_decode_attention(pool.handle, ids, q, w.scale, out, lse, ws, stream)
        if gather:
            gather(out, lse)

    if args.profile_steps:
        for _ in range(args.profile_steps):
            step()
        torch.cuda.synchronize()
        return 0

    sampler = ClockSampler(local)
    sampler.start()   # before warm-up: nvidia-smi's start-up stays out of the timed region
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = pool.last_launch_count()
    decode_path = pool.last_decode_path()
    kernel_cfg = pool.last_kernel_config()
    sampler.mark()
    pool.set_profiling(True)
    pool.kernel_times()  # clear
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    for i in range(args.steps):
        step()
        evs[i + 1].record(stream)   # per-step boundaries (for percentiles; no sync inside)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    kt = pool.kernel_times()
    pool.set_profiling(False)
    ms = evs[0].elapsed_time(evs[-1]) / args.steps
    per_step_raw = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    per_step = sorted(per_step_raw)
    pct = {"p10": per_step[int(0.1 * (len(per_step) - 1))], "p50": statistics.median(per_step),
           "p90": per_step[int(0.9 * (len(per_step) - 1))], "max": per_step[-1],
           "max_step": per_step_raw.index(per_step[-1])}
    ms = max_over_ranks(ms, world, "cuda")
    n_total = len(w0.n) if args.strong else world * n_req
    value = n_total / (ms / 1e3)

    # ---- CUDA-graph variant: one hc_decode_attention call (descriptor H2D
    # copy from the runtime's pinned staging buffer + kernels) captured once and replayed —
    # valid while the batch (ids, cache contents) is fixed, as in this loop; kernel-side
    # work is identical, only host launch overhead goes away.
    graph = None
    if world == 1 and not args.no_graph:
        try:
            gr = torch.cuda.CUDAGraph()
            torch.cuda.synchronize()
            with torch.cuda.graph(gr, capture_error_mode="relaxed"):
                hc.hc_decode_attention(pool.handle, ids, q, w.scale, out, lse, ws, torch.cuda.current_stream())
            for _ in range(2):
                gr.replay()
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            for _ in range(args.steps):
                gr.replay()
            g1.record()
            torch.cuda.synchronize()
            ms_g = g0.elapsed_time(g1) / args.steps
            graph = {"value": n_total / (ms_g / 1e3), "unit": "req-layers/s", "ms_per_step": ms_g,
                     "note": "one decode call captured as a CUDA graph and replayed (fixed batch)"}
            del gr
        except Exception as ex:   # report, never fall back silently
            graph = {"error": f"{type(ex).__name__}: {ex}"[:300]}

    # ---- end to end through the public API: pinned host q -> device, decode, out + lse -> host,
    # every step.  As a serving loop would, the copies run on their own stream, double-buffered:
    # step i+1's q upload and step i-1's read-back overlap step i's decode.
    e2e = None
    if not args.no_e2e:
        q_host = [q.cpu().pin_memory() for _ in range(2)]
        out_host = [torch.empty(out.shape, dtype=out.dtype).pin_memory() for _ in range(2)]
        lse_host = [torch.empty(lse.shape, dtype=lse.dtype).pin_memory() for _ in range(2)]
        q_dev = [torch.empty_like(q) for _ in range(2)]
        o_dev = [torch.empty_like(out) for _ in range(2)]
        l_dev = [torch.empty_like(lse) for _ in range(2)]
        cs, ds = torch.cuda.Stream(), torch.cuda.Stream()   # uploads / read-backs (in-order each)
        up = [torch.cuda.Event() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        back = [torch.cuda.Event() for _ in range(2)]

        def e2e_steps(n):
            for i in range(n):
                b = i & 1
                with torch.cuda.stream(cs):
                    if i >= 2:
                        cs.wait_event(back[b])   # host buffers / device q of step i-2 are free
                    q_dev[b].copy_(q_host[b], non_blocking=True)
                    up[b].record(cs)
                stream.wait_event(up[b])
                if i >= 2:
                    stream.wait_event(back[b])   # o_dev[b], l_dev[b] read back already
                hc.hc_decode_attention(pool.handle, ids, q_dev[b], w.scale, o_dev[b], l_dev[b], ws, stream)
                done[b].record(stream)
                with torch.cuda.stream(ds):
                    ds.wait_event(done[b])
                    out_host[b].copy_(o_dev[b], non_blocking=True)
                    lse_host[b].copy_(l_dev[b], non_blocking=True)
                    back[b].record(ds)

        e2e_steps(4)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        cs.wait_event(f0)
        ds.wait_event(f0)
        e2e_steps(args.steps)
        f1.record(ds)   # after the last read-back
        torch.cuda.synchronize()
        assert torch.equal(out_host[(args.steps - 1) & 1].cuda(), out), "e2e result differs from the device-timed loop"
        ms_e2e = max_over_ranks(f0.elapsed_time(f1) / args.steps, world, "cuda")
        e2e = {"value": n_total / (ms_e2e / 1e3), "unit": "req-layers/s",
               "h2d_bytes_per_step": q.numel() * q.element_size(),
               "d2h_bytes_per_step": out.numel() * out.element_size() + lse.numel() * lse.element_size(),
               "ms_per_step": ms_e2e,
               "note": "pinned host q -> device, hc_decode_attention, out + lse -> pinned host every step; "
                       "uploads and read-backs on their own streams, double-buffered across steps"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peaks, peak_src = load_peaks()
    B_alg, F_alg, kv_tok, hid_tok = algorithmic(w)
    calls = max(1, kt["calls"])
    t_rec, t_att, t_comb, t_up = (kt["recon_ms"] / calls, kt["attn_ms"] / calls, kt["combine_ms"] / calls,
                                  kt["upload_ms"] / calls)
    d, s = w.shape.d, w.elem_bytes
    hbm = peaks["hbm_gbs"]
    tf_burst, tf_sus = peaks["bf16_tflops"], peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    # the sustained (power-capped) peak for a step that ran capped, the burst peak when the
    # SM clock held its maximum through the timed region (B200_PROFILING: burst vs sustained)
    # A power-cap flag counts only when the timed region lasted long enough (>= 1 s) to
    # reach the capped steady state the sustained figure was measured in (4 s back to
    # back); a short region at a held clock is a burst.
    timed_s = ms * args.steps / 1e3
    capped = not clocks or clocks.get("sm_mhz", 0) < 0.90 * (clocks.get("sm_max_mhz") or 1e9) \
        or ("sw_power_cap" in clocks.get("reasons", []) and timed_s >= 1.0)
    tf_peak = tf_sus if capped else tf_burst
    tf_kind = ("bf16 sustained (power-capped run), " if capped else "bf16 burst (clock held max), ") + peak_src
    fused = decode_path == 1
    absorbed = decode_path == 3
    if absorbed:
        n_h = sum(1 for m in w.modes if m == 1)
        ab_bytes = 2 * hid_tok * d * s + 2 * d * d * s + 4 * n_h * d * 2 * 2
        # the variant's own floor: x read twice (scores, then Z), W_K and W_V once, q/out
        B_alg = kv_tok * 2 * d * s + 2 * hid_tok * d * s + 2 * d * d * s + 2 * n_req * d * s
        F_alg = 0
    kernels = {
        ("fused_step" if fused else "recon_gemm"): {
            "ms": t_rec, "bound": "tensor", "unit": "TFLOP/s",
            "achieved": (F_alg / (t_rec / 1e3) / 1e12) if t_rec > 0 else None, "flops_per_launch": F_alg,
            "note": "GEMM + split-K attention warps in one kernel; FLOP/s counts the GEMM only" if fused else ""},
        "attention": ({"ms": None, "note": "n/a: the attention runs inside fused_step_kernel"} if fused else
                      {"ms": t_att, "bound": "hbm", "unit": "GB/s",
                       "bytes_per_launch": (kv_tok + hid_tok) * 2 * w.shape.dk * s,
                       "achieved": ((kv_tok + hid_tok) * 2 * w.shape.dk * s / (t_att / 1e3) / 1e9) if t_att > 0 else None}),
        "combine": {"ms": t_comb},
        "descriptor_upload": {"ms": t_up},
    }
    if absorbed:
        del kernels["recon_gemm"]
        kernels["attention"]["bytes_per_launch"] = kv_tok * 2 * d * s
        kernels["attention"]["achieved"] = (kv_tok * 2 * d * s / (t_att / 1e3) / 1e9) if t_att > 0 else None
        kernels["absorbed_hidden"] = {
            "ms": t_rec, "bound": "hbm", "unit": "GB/s", "bytes_per_launch": ab_bytes,
            "achieved": (ab_bytes / (t_rec / 1e3) / 1e9) if t_rec > 0 else None,
            "note": "5 kernels: q~, scores, Z and W_V GEMMs on tcgen05, P rescale; bytes = x read twice + W_K + W_V + q~/Z round trips"}
        dom = "absorbed_hidden" if t_rec >= t_att else "attention"
    else:
        dom = ("fused_step" if fused else "recon_gemm") if (fused or t_rec >= t_att) else "attention"
    k = kernels[dom]
    if dom == "absorbed_hidden":
        roof = {"bound": "hbm", "kernel": "absorbed qt/score/rescale/z/wv kernels", "achieved": k["achieved"],
                "peak": hbm, "unit": "GB/s", "frac": k["achieved"] / hbm, "traffic": None,
                "peak_kind": "HBM copy, " + peak_src}
    elif dom != "attention":
        peak = tf_peak
        if k["achieved"] > tf_sus and peak == tf_sus:
            # faster than the capped steady state: the clock dipped below 90% of max without the
            # cap binding, so the burst peak is the honest denominator (never report frac > 1)
            peak, tf_kind = tf_burst, "bf16 burst (achieved exceeds the sustained figure), " + peak_src
        fcfg = str(kernel_cfg % 10000)
        fname = (f"fused_step_kernel<{fcfg[0]},{fcfg[1]},{fcfg[2]}" + (f",+{fcfg[3]} epilogue warps" if len(fcfg) > 3 else "")
                 + (", 256x256 tiles" if kernel_cfg >= 10000 else "") + ">")
        roof = {"bound": "tensor", "kernel": fname if fused else "recon_tc2_kernel<2,4>",
                "achieved": k["achieved"], "peak": peak,
                "unit": "TFLOP/s", "frac": k["achieved"] / peak,
                "frac_vs_burst": k["achieved"] / tf_burst, "frac_vs_sustained": k["achieved"] / tf_sus,
                "traffic": TRAFFIC.get(w.name, {}).get(dom),
                "ncu_tensor_pipe_pct": TRAFFIC.get(w.name, {}).get(dom + "_tensor_pipe_pct"),
                "peak_kind": tf_kind}
    else:
        peak = hbm
        roof = {"bound": "hbm", "kernel": "attn_pipe_kernel<128,8,3>", "achieved": k["achieved"], "peak": peak,
                "unit": "GB/s", "frac": k["achieved"] / peak, "traffic": TRAFFIC.get(w.name, {}).get("attention"),
                "peak_kind": "HBM copy, " + peak_src}
    # the step's own FLOP rate above the sustained figure means it never reached the capped
    # steady state: bound it by the burst peak (T_roof / T stays <= 1 for a tensor-bound step)
    tf_step = tf_burst if (tf_peak == tf_sus and ms > 0 and F_alg / (ms * 1e-3) / 1e12 > tf_sus) else tf_peak
    T_roof = max(F_alg / (tf_step * 1e12), B_alg / (hbm * 1e9))
    line = {
        "metric": METRIC, "value": value, "unit": "req-layers/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "step_ms_percentiles": pct, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None, "dtype": "bf16" if w.dtype == "bf16" else "f32", "data": "synthetic",
        "config": {"workload": w.name, "shape": w.shape.name, "d": d, "heads": w.shape.H, "head_dim": w.shape.dh,
                   "kv_heads": w.shape.n_kv,
                   "cache_bytes_per_token": {"kv": 2 * w.shape.dk * s, "hidden": d * s,
                                             "hidden_over_kv": d / (2 * w.shape.dk)},
                   "block_size": w.block_size, "n_req_per_gpu": n_req, "kv_tokens": kv_tok, "hidden_tokens": hid_tok,
                   "hidden_request_frac": sum(w.modes) / n_req, "parallelism": f"request-sharded x{world} ({'strong, LPT' if args.strong else 'weak'})",
                   "output_gather": gather.describe() if gather else "none",
                   "l2": "inputs larger than L2 (whole cache read every step)", "note": w.note,
                   "fill": args.fill,
                   "variant": "absorbed hidden attention (NON-PAPER, HC_FLAG_ABSORB_HIDDEN)" if absorbed
                   else "paper (hidden K/V rebuilt every step)",
                   "rope_theta": args.rope},
        "roofline": roof,
        "step_roofline": {"T_roof_ms": T_roof * 1e3, "frac": T_roof * 1e3 / ms, "alg_bytes": B_alg,
                          "alg_flops": F_alg, "alg_GBps": B_alg / (ms / 1e3) / 1e9,
                          "alg_TFLOPs": F_alg / (ms / 1e3) / 1e12, "peaks": peak_src},
        "kernels": kernels,
        "gpu_launches": launches_per_step * args.steps,
        "e2e": e2e,
        "cuda_graph": graph,
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_module_mode(args, rank, world, local):
    """--mode layer / prefill: the attention-module rows f1 / f3 (not the north-star line)."""
    import torch

    from paper_2504_07494_b200 import build as hb
    hb.build()
    from paper_2504_07494_b200 import hc
    from synth import configs as C
    from synth import drive as T
    from synth.configs import Workload

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w0 = workload_from(args.config)
    d = w0.shape.d
    peaks, peak_src = load_peaks()
    tf = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    if args.mode == "layer":
        w = w0
        pool = T.make_layer_pool(w, device=local)
        T.fill(pool, T.prefix_workload(w), device=local)
        x = torch.stack([w.x_t(i, device=dev) for i in range(len(w.n))]).contiguous()
        ids, modes = list(w.req_ids), list(w.modes)
        y = torch.empty_like(x)
        lse = torch.empty((len(ids), w.shape.H), dtype=torch.float32, device=dev)
        # contexts grow by one token per step: leave room for the growth of the split/scratch plan
        ws_need = hc.hc_layer_workspace_size(pool.handle, ids, modes)
        ws = torch.empty(int(ws_need * 1.05) + (8 << 20), dtype=torch.uint8, device=dev)
        n_layer = len(ids)

        def step():
            # one decode layer per step: the cache grows by one token per request, so free the
            # token again by re-running on a pool snapshot is not possible; instead measure
            # consecutive steps (contexts grow by 1 token per step, < 0.1% over the run)
            hc.hc_decode_layer(pool.handle, ids, modes, x, w.scale, y, lse, ws)
        hid = w.n_tokens(1) + args.warmup + args.steps
        flops = 4 * d * d * w.n_tokens(1) + 2 * len(ids) * d * 3 * d + 2 * len(ids) * d * d
        unit, metric = "req-layers/s", "decode-layer req-layers/s (q/k/v proj + cache write, attention, W_O)"
    else:
        L, nreq = args.prefill_len, args.prefill_reqs
        w = Workload(f"prefill-{w0.shape.name}-{nreq}x{L}", w0.shape, w0.block_size, w0.dtype, 21, [L] * nreq,
                     [i % 2 for i in range(nreq)], list(range(nreq)))
        pool = T.make_layer_pool(w, device=local, num_blocks=T.pool_blocks(w) * (args.warmup + args.steps + 1))
        x = torch.cat([w.x(i, device=dev) for i in range(nreq)]).contiguous()
        y = torch.empty_like(x)
        state = {"k": 0}

        def step():
            base = 1_000_000 * (state["k"] + 1)
            state["k"] += 1
            pool.prefill_layer([base + r for r in w.req_ids], w.modes, w.n, x, w.scale, y=y)
        flops = 8 * nreq * L * d * d + 2 * nreq * L * L * d
        n_layer = nreq * L
        unit, metric = "tokens/s", "prefill-layer tokens/s (projections + causal attention + W_O)"
    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    time.sleep(0.3)
    sampler.mark()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    # A power-cap flag counts only when the timed region lasted long enough (>= 1 s) to
    # reach the capped steady state the sustained figure was measured in (4 s back to
    # back); a short region at a held clock is a burst.
    timed_s = ms * args.steps / 1e3
    capped = not clocks or clocks.get("sm_mhz", 0) < 0.90 * (clocks.get("sm_max_mhz") or 1e9) \
        or ("sw_power_cap" in clocks.get("reasons", []) and timed_s >= 1.0)
    peak = tf if capped else peaks["bf16_tflops"]
    achieved = flops / (ms / 1e3) / 1e12
    line = {"metric": metric, "mode": args.mode, "value": n_layer / (ms / 1e3), "unit": unit, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "dtype": w.dtype, "data": "synthetic", "config": {"workload": w.name, "d": d},
            "roofline": {"bound": "tensor", "kernel": "whole layer (projection GEMMs + attention)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "flops_per_step": flops,
                         "peak_kind": ("bf16 sustained (power-capped run), " if capped
                                       else "bf16 burst (clock held max), ") + peak_src},
            "tensor_TFLOPs": achieved, "frac_of_sustained_bf16": achieved / tf,
            "gpu_launches_per_step": pool.last_launch_count(),
            "gpu_launches": pool.last_launch_count() * args.steps, "clocks": clocks}
    print(json.dumps(line), flush=True)
    return 0


# ncu --set full per-launch DRAM traffic (bytes) of the dominant kernels, from the
# committed profiles/ summaries; None until measured.
TRAFFIC = {}
_tp = os.path.join(ROOT, "profiles", "traffic.json")
if os.path.exists(_tp):
    try:
        TRAFFIC = json.load(open(_tp))
    except Exception:
        TRAFFIC = {}

if __name__ == "__main__":
    sys.exit(main())
