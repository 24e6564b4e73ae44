"""Host wall-clock breakdown of one bench step (create / levelize / run_batch / close)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hfgen
from paper_2203_08395_b200 import hf
dev = torch.device("cuda:0")
g = hfgen.config("C4")
S = 64
D = torch.from_numpy(hfgen.scenario_delays(g, 0, S, "ms")).to(dev)
T = torch.full((S,), g.t_req, dtype=torch.float32, device=dev)
in_ptr = torch.from_numpy(g.in_ptr).to(dev); in_src = torch.from_numpy(g.in_src).to(dev)
delay = torch.from_numpy(g.delay).to(dev); at_src = torch.from_numpy(g.at_src).to(dev)
w = torch.empty(S, dtype=torch.float32, device=dev)
st = torch.cuda.current_stream()
prof = "--prof" in sys.argv
flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size // 4, dtype=torch.float32, device=dev) if "--flush" in sys.argv else None
import contextlib
cm = contextlib.nullcontext()
if "--sampler" in sys.argv or "--smi" in sys.argv:
    import bench
    if "--smi" in sys.argv:
        import sys as _s
        _s.modules["pynvml"] = None   # force the nvidia-smi fallback
    cm = bench.ClockSampler(0)
cm.__enter__()
for it in range(int(os.environ.get("ITERS", "8"))):
    if flush is not None:
        flush.fill_(1.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G = hf.hf_graph_create(g.n, g.m, in_ptr, in_src, delay=delay, stream=st)
    if prof:
        hf.hf_profile_enable(G, True)
    t1 = time.perf_counter()
    hf.hf_levelize(G)
    t2 = time.perf_counter()
    hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, at_src, w)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    if prof:
        hf.hf_profile_read(G)
    t4 = time.perf_counter()
    G.close()
    t5 = time.perf_counter()
    print(f"create {1e3*(t1-t0):7.2f}  levelize {1e3*(t2-t1):7.2f}  run_batch(enqueue) {1e3*(t3-t2):7.2f}  sync {1e3*(t4-t3):7.2f}  close {1e3*(t5-t4):7.2f}  total {1e3*(t5-t0):7.2f} ms", flush=True)
cm.__exit__(None, None, None)
if hasattr(cm, "summary"):
    print(cm.summary())
