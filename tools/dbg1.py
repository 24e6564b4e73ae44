import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import hfgen, oracle
from paper_2203_08395_b200 import hf
dev = torch.device("cuda:0")
g = hfgen.config("C1")
G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev), torch.from_numpy(g.in_src).to(dev), delay=torch.from_numpy(g.delay).to(dev), stream=torch.cuda.current_stream())
L = hf.hf_levelize(G)
print("L", L, flush=True)
at = torch.empty(g.n, dtype=torch.float32, device=dev)
hf.hf_propagate_forward(G, torch.from_numpy(g.at_src).to(dev), at)
torch.cuda.synchronize()
print("fwd ok", flush=True)
