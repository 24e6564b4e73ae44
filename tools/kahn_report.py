import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 3).astype(np.int64)
a = a[a[:, 0] > 0]
t0, t1, sz = a.T
work = t1 - t0
bar = t0[1:] - t1[:-1]
print(f"rounds {len(a)}, span {(t1[-1] - t0[0]) / 1e3:.1f} us; per round: expand median {np.median(work) / 1e3:.2f} us "
      f"(max {work.max() / 1e3:.2f}), barrier median {np.median(bar) / 1e3:.2f} us; frontier median {np.median(sz):.0f} max {sz.max()}")
