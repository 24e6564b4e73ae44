import sys, os, ctypes, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2203_08395_b200 import hf
dev = torch.device("cuda:0")
G = hf.hf_graph_create(2, 1, torch.tensor([0, 0, 1], dtype=torch.int32, device=dev), torch.tensor([0], dtype=torch.int32, device=dev), stream=torch.cuda.current_stream())
lib = hf._lib
lib.hf_debug_scan.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
rng = np.random.default_rng(0)
bad = 0
for it, n in enumerate([1, 5, 4095, 4096, 4097, 10001, 100000, 1500001, 3, 2500000, 8191, 123457]):
    a = rng.integers(0, 10, n).astype(np.int32)
    x = torch.from_numpy(a).to(dev)
    y = torch.empty_like(x)
    tot = torch.zeros(1, dtype=torch.int32, device=dev)
    st = lib.hf_debug_scan(G.handle, x.data_ptr(), y.data_ptr(), n, tot.data_ptr())
    ref = np.concatenate([[0], np.cumsum(a)[:-1]]).astype(np.int64)
    got = y.cpu().numpy().astype(np.int64)
    ok = np.array_equal(ref, got) and int(tot.item()) == int(a.sum())
    if not ok:
        bad += 1
        i = int(np.argmax(ref != got)) if not np.array_equal(ref, got) else -1
        print(f"n={n} MISMATCH st={st} first bad {i} ref {ref[i] if i>=0 else None} got {got[i] if i>=0 else None} tot {tot.item()} vs {a.sum()}")
    else:
        print(f"n={n} ok")
print("bad", bad)
