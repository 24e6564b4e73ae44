#!/usr/bin/env python
"""Benchmark: DAG propagation edges/s (fwd+bwd) on B200, % of HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hf|reference]
                    [--config C4|C1|C2-chain|C2-tree|C2-random|C3|C5]
                    [--scenarios S] [--scaling strong|weak]

`--gpus N` runs N ranks: under torchrun (RANK / WORLD_SIZE set by the launcher) or,
when started directly, by re-launching itself through torch.distributed.run with N
processes (one per GPU, 127.0.0.1 rendezvous).

Default workload (BASELINE.json:10, config C4): the 1.5M-pin / 2.5M-arc circuit-shaped
timing DAG (levelized generator, D = 200, seed 4) with 64 what-if delay scenarios
split over the N ranks (strong scaling; `--scaling weak` gives 64 per rank).  The
graph is created and levelized once, before the timed region (the levelization is
timed on its own and reported in `phases_ms.levelize` and `full_step`).  One step =
  hf_run_batch_d (forward + backward + slack + worst slack for the rank's scenarios)
  -> NCCL all-gather of the worst slacks (N > 1)
on device-resident inputs.  value = 2*m*S_total / t_step (max over ranks), L2 flushed
(a 2x L2 write) before every timed step, and the inputs exceed L2.

Other configs (one bench line each, same contract):
  C1        forward only (BASELINE.json:7), value = m / t_fwd
  C2-*      levelization (BASELINE.json:8), value = m / t_levelize
  C3, C5    single delay set, forward + backward + worst slack (BASELINE.json:9, 11)
Single-graph configs do not shard: at N > 1 every rank runs a replica ("replicas
only", value summed over ranks).

e2e = the same metric through the host-pointer C ABI: the step's inputs go up from
pinned host memory and the result comes back inside the timed region.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import hfgen  # noqa: E402

METRIC = "DAG propagation edges/sec (fwd+bwd) at 1/2/4/8 B200; % HBM roofline"
UNIT = "edges/s"
# the paper's only speed-up claim, on its own workload
PAPER_CONTEXT = {
    "speedup": 7.7,
    "what": "Heteroflow timing-analysis task graph, 99 min (1 core + 1 GPU) vs 13 min "
            "(40 cores + 4 GPUs), RTX 2080, netcard 1024 views (PAPER.md:38-40, 1103-1106)",
    "comparable": False,
}
KINDS = {"C1": "forward", "C2-chain": "levelize", "C2-tree": "levelize",
         "C2-random": "levelize", "C3": "single", "C4": "batch", "C5": "single"}


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="hf", choices=["hf", "reference"])
    p.add_argument("--config", default="C4", choices=sorted(KINDS))
    p.add_argument("--scenarios", type=int, default=64,
                   help="batch configs: scenarios in total (strong) or per rank (weak)")
    p.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-secondary", action="store_true",
                   help="skip the full-step / weak-scaling secondary measurements")
    p.add_argument("--ncu", action="store_true", help="short run for an ncu capture (no timing)")
    p.add_argument("--dry-run", action="store_true",
                   help="launcher check without a GPU: ranks rendezvous over gloo and rank 0 "
                        "prints the line skeleton")
    return p.parse_args(argv)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args):
    """`--gpus N` started directly (no WORLD_SIZE): re-run as N ranks under
    torch.distributed.run and exit with its status."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))


def scenario_block(args, rank, world):
    from paper_2203_08395_b200.shard import scenario_block as blk
    return blk(rank, world, args.scenarios, args.scaling)


def algorithmic_bytes(n, m, S):
    """bytes the method must move per fwd / bwd pass."""
    b_fwd = (4 * (n + 1) + 4 * m + 4 * n) + S * (4 * m + 4 * n + 4 * n)
    b_bwd = (4 * (n + 1) + 4 * m + 4 * m + 4 * n) + S * (4 * m + 4 * n + 4 * n + 4 * n) + 4 * S
    return b_fwd, b_bwd


def levelize_bytes(n, m):
    """B_lev = 4(n+1) + 4m + 8n (cnt RMW) + 4n (level) + 4n (order)."""
    return 4 * (n + 1) + 4 * m + 8 * n + 4 * n + 4 * n


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled (in-process NVML, every 2 ms) during the
    timed region; nvidia-smi every 200 ms is the fallback."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    _nvml = None   # (module, handle, reasons fn, sm max, mem max) per process, set up once

    def __init__(self, index: int, period: float = 0.002):
        self.index = index
        self.period = period
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        # NVML init and the handle lookup take ~0.1 s: done here, before the timed
        # region, so the sampling thread starts sampling at once (round 1 got 1-4
        # samples per run because nvmlInit ran inside the timed region)
        if ClockSampler._nvml is None and not os.environ.get("HF_BENCH_NO_CLOCKS"):
            try:
                import pynvml as nv
                nv.nvmlInit()
                h = nv.nvmlDeviceGetHandleByIndex(index)
                getr = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                ClockSampler._nvml = (nv, h, getr, nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
                                      nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_MEM))
            except Exception:
                ClockSampler._nvml = False

    def _run(self):
        if os.environ.get("HF_BENCH_NO_CLOCKS"):   # diagnostics only
            return
        try:
            if not ClockSampler._nvml:
                raise RuntimeError("no NVML")
            nv, h, getr, mx, mmx = ClockSampler._nvml
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mem = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM)
                r = int(getr(h))
                act = lambda bit: "Active" if r & bit else "Not Active"
                self.rows.append([str(sm), str(mx), "", hex(r), act(0x8), act(0x40), act(0x20),
                                  act(0x4), str(mem), str(mmx)])
                self._stop.wait(self.period)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        mem = [float(r[8]) for r in self.rows if len(r) > 9 and r[8].isdigit()]
        mmx = [float(r[9]) for r in self.rows if len(r) > 9 and r[9].isdigit()]
        out = {"sm_mhz": float(np.median(sm)) if sm else None,
               "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
               "samples": len(self.rows)}
        if mem:   # HBM clock (box-to-box differences in memory bandwidth show here)
            out["mem_mhz"] = float(np.median(mem))
            out["mem_max_mhz"] = max(mmx) if mmx else None
        return out


def copy_probe(dev):
    """This box's device copy bandwidth (read + write bytes of a 2 GiB copy, best of 5,
    CUDA events), measured after the timed region: context for roofline.peak, which
    is the pool's MEASURED_PEAKS.json figure."""
    import torch
    try:
        a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
        b = torch.empty_like(a)
        best = None
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        del a, b
        return round(2 * (2 << 30) / (best * 1e-3) / 1e9, 1)
    except Exception:
        return None


# ---- the oracle (cpu_baseline of the GPU arm, and the whole reference arm) -------------
def oracle_step(kind, g, D=None, T=None, threads=1):
    """One pass of the config's work by the CPU oracle; returns the edges it counts."""
    import oracle
    if kind == "batch":
        oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=threads)
        return 2 * g.m * D.shape[1]
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    if kind == "levelize":
        return g.m
    at = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, lv)
    if kind == "forward":
        return g.m
    oracle.backward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.t_req, at, lv)
    return 2 * g.m


def oracle_note(kind, cfg, S, threads):
    what = {"batch": f"levelize + fwd + bwd + wns for {S} scenarios, {threads} threads "
                     "(one std::thread per scenario)",
            "levelize": "FIFO Kahn levelization + canonical order, 1 thread",
            "forward": "levelize + forward, 1 thread",
            "single": "levelize + forward + backward + wns, 1 thread"}[kind]
    return f"{cfg}: oracle {what} (its levelization inside the timed pass)"


def cpu_baseline(kind, cfg, g, D, T):
    cores = os.cpu_count() or 1
    threads = cores if kind == "batch" else 1
    t0 = time.perf_counter()
    edges = oracle_step(kind, g, D, T, threads)
    dt = time.perf_counter() - t0
    return {"value": edges / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": oracle_note(kind, cfg, None if D is None else D.shape[1], threads) +
            ", one pass of the full workload", "seconds": round(dt, 3)}


def workload(args, g, kind, S, S_total, world):
    name = args.config
    if kind == "batch":
        w = (f"{name}: levelized circuit DAG n={g.n} m={g.m} D={g.depth}, {S_total} what-if "
             f"scenarios ({S}/rank, {args.scaling} scaling); step = hf_run_batch_d fwd+bwd+wns "
             f"+ NCCL gather of worst slack on a graph levelized before the timed region")
    elif kind == "levelize":
        w = f"{name}: n={g.n} m={g.m}; step = hf_levelize (levels, canonical order, relabel)"
    elif kind == "forward":
        w = (f"{name}: levelized circuit DAG n={g.n} m={g.m} D={g.depth}; step = "
             f"hf_propagate_forward_d (one delay set)")
    else:
        w = (f"{name}: n={g.n} m={g.m}; step = hf_propagate_forward_d + hf_propagate_backward_d "
             f"(one delay set, slack + worst slack) on a levelized graph")
    return {"workload": w, "n": g.n, "m": g.m, "levels": g.depth, "scenarios_per_gpu": S,
            "scenarios_total": S_total,
            "parallelism": (f"scenario-shard x{world}" if kind == "batch"
                            else f"replicas x{world}"),
            "l2": "flushed between steps (2x L2 write) and inputs > L2"}


def run_reference(args):
    """The oracle as the reference arm (this tier has no installable reference): each
    step one bounded sample of the config's workload on the host cores."""
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return
    kind = KINDS[args.config]
    g = hfgen.config(args.config)
    world = max(ws, args.gpus)
    S_total = args.scenarios * (world if args.scaling == "weak" else 1)
    S = args.scenarios if args.scaling == "weak" else args.scenarios // world
    D = T = None
    cores = os.cpu_count() or 1
    threads = 1
    if kind == "batch":
        S_ref = min(8, S)   # bounded sample: a few scenarios per step
        D = hfgen.scenario_delays(g, 0, S_ref, "ms")
        T = np.full(S_ref, g.t_req, np.float32)
        threads = cores
    for _ in range(args.warmup):
        oracle_step(kind, g, D, T, threads)
    t0 = time.perf_counter()
    edges = 0
    for _ in range(args.steps):
        edges += oracle_step(kind, g, D, T, threads)
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    v = edges / max(args.steps, 1) / dt
    sample = oracle_note(kind, args.config, None if D is None else D.shape[1], threads)
    if kind == "batch":
        sample += f" -- a bounded sample: {D.shape[1]} of the {S} scenarios per step"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": args.scaling if kind == "batch" else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload(args, g, kind, S if kind == "batch" else 1,
                               S_total if kind == "batch" else world, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "paper_context": PAPER_CONTEXT}
    print(json.dumps(line), flush=True)


def dry_run(args):
    """Launcher check without a GPU: all ranks rendezvous over gloo, rank 0 prints."""
    import torch
    import torch.distributed as dist
    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.ones(1)
    if world > 1:
        dist.all_reduce(t)
    if world != args.gpus or int(t.item()) != world:
        raise SystemExit(f"world size {world} (ranks seen {t.item()}) != --gpus {args.gpus}")
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world,
                          "ranks_seen": int(t.item())}), flush=True)
    if world > 1:
        dist.destroy_process_group()


class Timer:
    """CUDA events on the launching stream around each timed step; the L2 is flushed
    (untimed) before every step."""

    def __init__(self, torch, stream, flush):
        self.torch, self.stream, self.flush = torch, stream, flush
        self.ms = []

    def step(self, fn):
        torch = self.torch
        self.flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        fn()
        e1.record(self.stream)
        e1.synchronize()
        self.ms.append(e0.elapsed_time(e1))


def max_over_ranks(torch, dist, dev, world, vals):
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    maybe_spawn(args)
    if args.dry_run:
        dry_run(args)
        return
    import torch
    import torch.distributed as dist
    from paper_2203_08395_b200 import hf

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"world size {world} != --gpus {args.gpus}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    kind = KINDS[args.config]
    g = hfgen.config(args.config)
    n, m = g.n, g.m
    K = max(args.steps, 1)

    # inputs resident in HBM before the timed region
    in_ptr = torch.from_numpy(g.in_ptr).to(dev)
    in_src = torch.from_numpy(g.in_src).to(dev)
    delay = torch.from_numpy(g.delay).to(dev)
    at_src = torch.from_numpy(g.at_src).to(dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4 + 1024, dtype=torch.float32, device=dev)
    comm = None
    if world > 1 and kind == "batch":
        uid = [hf.hf_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = hf.hf_nccl_comm_init(uid[0], rank, world, local)

    S, S_total = 1, world
    D_host = T_host = None
    if kind == "batch":
        s_lo, s_hi = scenario_block(args, rank, world)
        S = s_hi - s_lo
        S_total = S * world if args.scaling == "weak" else args.scenarios
        D_host = hfgen.scenario_delays(g, s_lo, s_hi, "ms")
        T_host = np.full(S, g.t_req, np.float32)

    # the graph: created and levelized before the timed region (C2: levelize is the step)
    G = hf.hf_graph_create(n, m, in_ptr, in_src, delay=delay, device=local, stream=stream)
    hf.hf_profile_enable(G, True)
    hf.hf_levelize(G)
    L = G.num_levels

    stats = {"fwd": 0.0, "bwd": 0.0, "phase": 0.0, "lev": 0.0, "launches": 0}
    if kind == "batch":
        D = torch.from_numpy(D_host).to(dev)
        T = torch.from_numpy(T_host).to(dev)
        wns = torch.empty(S, dtype=torch.float32, device=dev)
        wns_all = torch.empty(S * world, dtype=torch.float32, device=dev)

        def work():
            hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, at_src, wns, comm,
                            wns_all if comm else None)
    elif kind == "levelize":
        def work():
            hf.hf_levelize(G)
    else:
        at = torch.empty(n, dtype=torch.float32, device=dev)
        rat = torch.empty(n, dtype=torch.float32, device=dev)
        w1 = torch.empty(1, dtype=torch.float32, device=dev)

        def work():
            hf.hf_propagate_forward(G, at_src, at)
            if kind == "single":
                hf.hf_propagate_backward(G, float(g.t_req), at, rat, None, w1)

    def record():
        lev, fwd, bwd, k = hf.hf_profile_read(G)
        stats["lev"] += lev
        stats["fwd"] += fwd
        stats["bwd"] += bwd
        stats["phase"] += hf.hf_profile_read_batch(G) if kind == "batch" else fwd + bwd
        return k

    if args.ncu:
        for _ in range(max(args.warmup, 1) + K):
            work()
        torch.cuda.synchronize()
        return

    for _ in range(args.warmup):
        work()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    timer = Timer(torch, stream, flush)
    gc.collect()
    gc.disable()   # no collector pause inside the timed region
    with ClockSampler(local) as clk:
        k0 = hf.hf_profile_read(G)[3]
        for _ in range(K):
            timer.step(work)
            record()
        launches = hf.hf_profile_read(G)[3] - k0
    gc.enable()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms, fwd_ms, bwd_ms, lev_ms, phase_ms = max_over_ranks(
        torch, dist, dev, world, [sum(timer.ms), stats["fwd"], stats["bwd"], stats["lev"],
                                  stats["phase"]])
    ms_step = total_ms / K
    peak, peak_src = peaks()

    # ---- metric and roofline of the dominant kernel(s)
    if kind == "batch":
        edges_step = 2.0 * m * S_total
        b_fwd, b_bwd = algorithmic_bytes(n, m, S)
        kern_ms = (fwd_ms + bwd_ms) / K
        algo = b_fwd + b_bwd
        kname = "forward + backward propagation kernels (k_flow, or k_wide on wide graphs)"
    elif kind == "single":
        edges_step = 2.0 * m * world
        b_fwd, b_bwd = algorithmic_bytes(n, m, 1)
        kern_ms = (fwd_ms + bwd_ms) / K
        algo = b_fwd + b_bwd
        kname = "forward + backward propagation kernels (k_flow; on wide graphs at S = 1 the level-synchronous k_wide3 with its init and finalisation)"
    elif kind == "forward":
        edges_step = 1.0 * m * world
        algo = algorithmic_bytes(n, m, 1)[0]
        kern_ms = fwd_ms / K
        kname = "forward propagation kernel (k_flow)"
    else:
        edges_step = 1.0 * m * world
        algo = levelize_bytes(n, m)
        kern_ms = lev_ms / K
        kname = "hf_levelize: all its launches (Kahn + contraction + sort + relabel)"
    value = edges_step / (ms_step * 1e-3)
    achieved = algo / (kern_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None, "kernel": kname,
            "algorithmic_bytes": algo, "peak_source": peak_src}
    if kind in ("batch", "single"):
        # the propagation phase: first launch to worst slacks, incl. sentinel fills,
        # task schedules, long-row finalisation (the events of hf_run_batch)
        roof["phase_frac"] = algo / ((phase_ms / K) * 1e-3) / 1e9 / peak
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath)).get(f"{args.config}/S{S}")
            if tj:
                roof["traffic"] = tj["traffic"]
                roof["traffic_source"] = tj.get("source")
        except Exception:
            pass
    roof["copy_gbs_this_box"] = copy_probe(dev)

    # levelization of this graph on its own (C2: that is the step)
    if kind != "levelize":
        lev_ms_each = []
        for _ in range(3):
            flush.fill_(1.0)
            hf.hf_levelize(G)
            lev_ms_each.append(hf.hf_profile_read(G)[0])
        lev_one = max_over_ranks(torch, dist, dev, world, [float(np.median(lev_ms_each))])[0]
    else:
        lev_one = lev_ms / K

    # ---- secondary: the whole hot path per step (create + levelize + batch) and, at
    # N > 1, weak scaling (64 scenarios per rank)
    secondary = {}
    if kind == "batch" and not args.no_secondary:
        def full():
            G2 = hf.hf_graph_create(n, m, in_ptr, in_src, delay=delay, device=local, stream=stream)
            hf.hf_levelize(G2)
            hf.hf_run_batch(G2, S, D, hf.HF_LAYOUT_MS, T, at_src, wns, comm,
                            wns_all if comm else None)
            full.g = G2
        t2 = Timer(torch, stream, flush)
        for i in range(min(K, 10) + 2):
            if i < 2:
                full()
                torch.cuda.synchronize()
            else:
                t2.step(full)
            full.g.close()
        fms = max_over_ranks(torch, dist, dev, world, [float(np.mean(t2.ms))])[0]
        secondary["full_step"] = {"ms_per_step": fms, "value": edges_step / (fms * 1e-3),
                                  "what": "create + levelize + run_batch (+ gather) per step"}
        if world > 1:
            Dw = torch.from_numpy(hfgen.scenario_delays(g, rank * args.scenarios,
                                                        (rank + 1) * args.scenarios, "ms")).to(dev)
            Tw = torch.full((args.scenarios,), float(g.t_req), dtype=torch.float32, device=dev)
            ww = torch.empty(args.scenarios, dtype=torch.float32, device=dev)
            wa = torch.empty(args.scenarios * world, dtype=torch.float32, device=dev)
            t3 = Timer(torch, stream, flush)
            for i in range(min(K, 10) + 2):
                fn = lambda: hf.hf_run_batch(G, args.scenarios, Dw, hf.HF_LAYOUT_MS, Tw, at_src,
                                             ww, comm, wa)
                if i < 2:
                    fn()
                    torch.cuda.synchronize()
                else:
                    t3.step(fn)
            wms = max_over_ranks(torch, dist, dev, world, [float(np.mean(t3.ms))])[0]
            secondary["weak"] = {"scenarios_per_gpu": args.scenarios, "ms_per_step": wms,
                                 "value": 2.0 * m * args.scenarios * world / (wms * 1e-3)}

    # ---- e2e through the host-pointer ABI (pinned host buffers, H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        h_at_src = pin(g.at_src)
        if kind == "batch":
            h_D, h_T = pin(D_host), pin(T_host)
            h_w = pin(np.zeros(S, np.float32))
            h_wall = pin(np.zeros(S * world, np.float32)) if comm else None

            def e2e_step():
                hf.hf_run_batch(G, S, h_D, hf.HF_LAYOUT_MS, h_T, h_at_src, h_w, comm, h_wall)
            h2d = 4 * m * S + 4 * S + 4 * n
            d2h = 4 * S + (4 * S * world if comm else 0)
        elif kind == "levelize":
            h_ptr, h_src = pin(g.in_ptr), pin(g.in_src)
            h_level, h_order = pin(np.zeros(n, np.int32)), pin(np.zeros(n, np.int32))
            h_lptr = pin(np.zeros(n + 1, np.int32))

            def e2e_step():
                G2 = hf.hf_graph_create(n, m, h_ptr, h_src, device=local, stream=stream)
                hf.hf_levelize(G2, h_level, h_lptr, h_order)
                G2.close()
            h2d = 4 * (n + 1) + 4 * m
            d2h = 4 * n + 4 * (L + 1) + 4 * n
        else:
            h_at, h_rat = pin(np.zeros(n, np.float32)), pin(np.zeros(n, np.float32))
            h_w1 = pin(np.zeros(1, np.float32))

            def e2e_step():
                hf.hf_propagate_forward(G, h_at_src, h_at)
                if kind == "single":
                    hf.hf_propagate_backward(G, float(g.t_req), h_at, h_rat, None, h_w1)
            h2d = 4 * n + (4 * n if kind == "single" else 0)
            d2h = 4 * n + (4 * n + 4 if kind == "single" else 0)
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        te = Timer(torch, stream, flush)
        for _ in range(K):
            te.step(e2e_step)
        e2e_ms = max_over_ranks(torch, dist, dev, world, [sum(te.ms)])[0] / K
        e2e = {"value": edges_step / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 4)}
        if kind == "batch" and comm is None and not args.no_secondary:
            # the whole path from host buffers in one call (create + levelize + batch)
            h_ptr, h_src, h_delay = pin(g.in_ptr), pin(g.in_src), pin(g.delay)
            fn = lambda: hf.hf_analyze(n, m, h_ptr, h_src, S, h_D, h_T, h_at_src, h_w,
                                       delay=h_delay, device=local, stream=stream)
            fn()
            tf = Timer(torch, stream, flush)
            for _ in range(min(K, 10)):
                tf.step(fn)
            fms = float(np.mean(tf.ms))
            e2e["full_hf_analyze"] = {"value": edges_step / (fms * 1e-3), "ms_per_step": fms,
                                      "h2d_bytes_per_step": h2d + 4 * (n + 1) + 8 * m}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(kind, args.config, g, D_host, T_host)

    if rank == 0:
        phases = {"levelize": lev_one}
        if kind in ("batch", "single"):
            phases.update({"propagation_phase": phase_ms / K, "forward_kernel": fwd_ms / K,
                           "backward_kernel": bwd_ms / K})
        elif kind == "forward":
            phases["forward_kernel"] = fwd_ms / K
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": (args.scaling if kind == "batch" else "weak"), "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": workload(args, g, kind, S, S_total, world),
            "phases_ms": phases,
            "roofline": roof,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "paper_context": PAPER_CONTEXT,
        }
        if kind in ("batch", "single"):
            line["propagation_edges_per_s"] = edges_step / ((fwd_ms + bwd_ms) / K * 1e-3)
        line.update(secondary)
        print(json.dumps(line), flush=True)
    G.close()
    if comm is not None:
        hf.hf_nccl_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
