#!/usr/bin/env python
"""Benchmark: DAG propagation edges/s (fwd+bwd) on B200, % of HBM roofline.

Workload (BASELINE.json:10, config C4): the 1.5M-pin / 2.5M-arc circuit-shaped
timing DAG (levelized generator, D = 200, seed 4) with 64 what-if delay scenarios
per GPU (weak scaling; --scaling strong splits 64 over the ranks as in C4).

One step = the whole hot path over one batch:
  hf_graph_create_d (validate CSR, derive fan-out)  ->  hf_levelize_d
  ->  hf_run_batch_d (forward + backward + slack + worst slack for S_local
      scenarios)  ->  NCCL all-gather of worst slack (N > 1).
value = 2*m*S_total / t_step, inputs resident in HBM when the timed region
starts; L2 flushed (write of 2x L2) between timed steps.  e2e = the same metric
through the host-pointer C ABI (hf_graph_create / hf_levelize / hf_run_batch) with
the H2D of CSR + delays from pinned memory and the D2H of the worst slacks inside
the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hf|reference]
"""
from __future__ import annotations

import argparse
import gc
import json
import os
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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="hf", choices=["hf", "reference"])
    p.add_argument("--config", default="C4")
    p.add_argument("--scenarios", type=int, default=64, help="scenarios per GPU (weak) or total")
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--ncu", action="store_true", help="short run for an ncu capture (no timing)")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def scenario_block(args, rank, world):
    from paper_2203_08395_b200.shard import scenario_block as blk
    return blk(rank, world, args.scenarios, args.scaling)


def algorithmic_bytes(n, m, S):
    """bytes the method must move per fwd / bwd pass."""
    b_fwd = (4 * (n + 1) + 4 * m + 4 * n) + S * (4 * m + 4 * n + 4 * n)
    b_bwd = (4 * (n + 1) + 4 * m + 4 * m + 4 * n) + S * (4 * m + 4 * n + 4 * n + 4 * n) + 4 * S
    return b_fwd, b_bwd


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 100 ms) during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        if os.environ.get("HF_BENCH_NO_CLOCKS"):   # diagnostics only
            return
        # in-process NVML (light); a spawned nvidia-smi contends for the driver lock
        # with the timed CUDA calls, so it is only the fallback
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            getr = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            mmx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_MEM)
            while not self._stop.is_set():
                # three cheap queries per sample, 100 ms apart: NVML calls take driver
                # locks that the timed CUDA calls also need
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mem = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM)
                r = int(getr(h))
                act = lambda bit: "Active" if r & bit else "Not Active"
                self.rows.append([str(sm), str(mx), "", hex(r), act(0x8), act(0x40), act(0x20),
                                  act(0x4), str(mem), str(mmx)])
                self._stop.wait(0.1)
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


def cpu_baseline(g, D_host, T, at_src, sample_note):
    import oracle
    cores = os.cpu_count() or 1
    S = D_host.shape[1]
    t0 = time.perf_counter()
    oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D_host, T, at_src, "ms", threads=cores)
    dt = time.perf_counter() - t0
    return {"value": 2.0 * g.m * S / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": sample_note, "seconds": round(dt, 3)}


def arm_config(args, g, S, S_total, world):
    """The workload both arms report (the reference arm times a bounded sample of it)."""
    return {"workload": f"{args.config}: levelized circuit DAG n={g.n} m={g.m} D={g.depth}, "
                        f"{S} scenarios/GPU, create+levelize+fwd+bwd+wns per step",
            "n": g.n, "m": g.m, "levels": g.depth, "scenarios_per_gpu": S,
            "scenarios_total": S_total, "parallelism": f"scenario-shard x{world}",
            "l2": "flushed between steps (2x L2 write) and inputs > L2"}


def run_reference(args):
    """The oracle as the reference arm (this tier has no installable reference)."""
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return
    import oracle
    g = hfgen.config(args.config)
    S_ref = 8
    D = hfgen.scenario_delays(g, 0, S_ref, "ms")
    T = np.full(S_ref, g.t_req, np.float32)
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=cores)
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    v = 2.0 * g.m * S_ref / dt
    sample = (f"{args.config}: n={g.n} m={g.m}, a bounded sample: {S_ref} of the scenarios per "
              f"step (value = 2*m*{S_ref} / step time), oracle levelize+fwd+bwd+wns, "
              f"{cores} threads")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": arm_config(args, g, args.scenarios if args.scaling == "weak"
                                 else args.scenarios // max(ws, 1),
                                 args.scenarios * (ws if args.scaling == "weak" else 1), ws),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    from paper_2203_08395_b200 import hf

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()

    g = hfgen.config(args.config)
    n, m = g.n, g.m
    s_lo, s_hi = scenario_block(args, rank, world)
    S = s_hi - s_lo
    S_total = S * world if args.scaling == "weak" else args.scenarios
    D_host = hfgen.scenario_delays(g, s_lo, s_hi, "ms")
    T_host = np.full(S, g.t_req, np.float32)

    # inputs resident in HBM before the timed region
    in_ptr = torch.from_numpy(g.in_ptr).to(dev)
    in_src = torch.from_numpy(g.in_src).to(dev)
    delay = torch.from_numpy(g.delay).to(dev)
    at_src = torch.from_numpy(g.at_src).to(dev)
    D = torch.from_numpy(D_host).to(dev)
    T = torch.from_numpy(T_host).to(dev)
    wns = torch.empty(S, dtype=torch.float32, device=dev)
    wns_all = torch.empty(S * world, dtype=torch.float32, device=dev)
    comm = None
    if world > 1:
        uid = [hf.hf_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = hf.hf_nccl_comm_init(uid[0], rank, world, local)

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4 + 1024, dtype=torch.float32, device=dev)

    stats = {"lev": 0.0, "fwd": 0.0, "bwd": 0.0, "prop": 0.0, "launches": 0}

    verbose = bool(os.environ.get("HF_BENCH_VERBOSE"))

    def step(record=False):
        h0 = time.perf_counter()
        G = hf.hf_graph_create(n, m, in_ptr, in_src, delay=delay, device=local, stream=stream)
        hf.hf_profile_enable(G, record)
        h1 = time.perf_counter()
        hf.hf_levelize(G)
        h2 = time.perf_counter()
        hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, at_src, wns, comm,
                        wns_all if comm else None)
        if verbose and record:
            print(f"host: create {1e3 * (h1 - h0):.2f} levelize {1e3 * (h2 - h1):.2f} "
                  f"run_batch {1e3 * (time.perf_counter() - h2):.2f} ms", file=sys.stderr)
        return G

    def finish(G, record):
        # after the step's end event: profile reads synchronise, graph teardown
        if record:
            lev, fwd, bwd, k = hf.hf_profile_read(G)
            stats["lev"] += lev
            stats["fwd"] += fwd
            stats["bwd"] += bwd
            stats["prop"] += hf.hf_profile_read_batch(G)
            stats["launches"] += k
        G.close()

    if args.ncu:
        for _ in range(max(args.warmup, 1) + max(args.steps, 1)):
            finish(step(), False)
        torch.cuda.synchronize()
        return

    for _ in range(args.warmup):
        finish(step(), False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = 0.0
    # no Python garbage collection inside the timed region (a collection pause would
    # leave the GPU idle between the step's host round trips)
    gc.collect()
    gc.disable()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)                       # L2 flush between timed steps (untimed)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            G = step(record=True)
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            finish(G, True)
            if os.environ.get("HF_BENCH_VERBOSE"):
                print(f"step {e0.elapsed_time(e1):.3f} ms", file=sys.stderr)
    gc.enable()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([total_ms, stats["fwd"], stats["bwd"], stats["lev"], stats["prop"]],
                     dtype=torch.float64,
                     device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, fwd_ms, bwd_ms, lev_ms, phase_ms = t.tolist()
    K = max(args.steps, 1)
    ms_step = total_ms / K
    value = 2.0 * m * S_total / (ms_step * 1e-3)

    # ---- roofline of the dominant kernels: the forward and backward propagation
    # kernels (events bracket exactly the two persistent launches); the batch phase
    # (first kernel -> worst slacks, incl. fills and long-row finalisation) is
    # reported beside it
    b_fwd, b_bwd = algorithmic_bytes(n, m, S)
    prop_ms = (fwd_ms + bwd_ms) / K
    achieved = (b_fwd + b_bwd) / (prop_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    box_gbs = copy_probe(dev)
    traffic = None   # measured dram bytes of the same two kernels (profiles/traffic.json)
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and S == 64:
        try:
            traffic = json.load(open(tpath)).get(args.config)
        except Exception:
            traffic = None

    # ---- e2e through the host-pointer ABI (pinned host buffers, H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
        h_ptr, h_src, h_delay = pin(g.in_ptr), pin(g.in_src), pin(g.delay)
        h_D, h_T, h_at = pin(D_host), pin(T_host), pin(g.at_src)
        h_w = pin(np.zeros(S, np.float32))
        h_wall = pin(np.zeros(S * world, np.float32)) if comm else None

        def e2e_step():
            if comm is None:
                # one call: create + levelize + batch, scenario upload overlapped
                hf.hf_analyze(n, m, h_ptr, h_src, S, h_D, h_T, h_at, h_w, delay=h_delay,
                              device=local, stream=stream)
                return
            G = hf.hf_graph_create(n, m, h_ptr, h_src, delay=h_delay, device=local, stream=stream)
            hf.hf_levelize(G)
            hf.hf_run_batch(G, S, h_D, hf.HF_LAYOUT_MS, h_T, h_at, h_w, comm, h_wall)
            G.close()

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e2e_ms = 0.0
        for _ in range(args.steps):
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            e1.synchronize()
            e2e_ms += e0.elapsed_time(e1)
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = te.item() / K
        h2d = 4 * (n + 1) + 4 * m + 4 * m + 4 * m * S + 4 * S + 4 * n
        d2h = 4 * S + (4 * S * world if comm else 0)
        e2e = {"value": 2.0 * m * S_total / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(e2e_ms, 4)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(g, D_host, T_host, g.at_src,
                           f"{args.config} full: n={n} m={m}, {S} scenarios, oracle "
                           "levelize + fwd + bwd + wns, one pass")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": arm_config(args, g, S, S_total, world),
            "phases_ms": {"levelize": lev_ms / K, "propagation_phase": phase_ms / K,
                          "forward_kernel": fwd_ms / K, "backward_kernel": bwd_ms / K,
                          "other": ms_step - (lev_ms + phase_ms) / K},
            "propagation_edges_per_s": 2.0 * m * S_total / (prop_ms * 1e-3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "forward + backward dataflow propagation kernels (k_flow)",
                         "algorithmic_bytes": b_fwd + b_bwd, "peak_source": peak_src,
                         "copy_gbs_this_box": box_gbs},
            "e2e": e2e,
            "gpu_launches": stats["launches"],
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        hf.hf_nccl_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
