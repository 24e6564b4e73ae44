"""Per-level timing of the level-synchronous S=1 pass (k_wide1) from an HF_TRACE dump:
header int32 {L, blocks}, then uint64 [2L][blocks] = per level and block {start (barrier
passed), its units done}.  Prints per level: level span (first start -> next level's
first start), median / max block busy time, and the barrier tail (last block done ->
next start).

    python tools/wide_trace.py c5_w1_fwd.bin [c5_w1_bwd.bin]
"""
import sys

import numpy as np


def main(fn):
    raw = open(fn, "rb").read()
    L, nb = np.frombuffer(raw[:8], dtype=np.int32)
    t = np.frombuffer(raw[8:], dtype=np.uint64).astype(np.int64).reshape(2 * L, nb)
    st, dn = t[0::2], t[1::2]
    t0 = st[0].min()
    print(f"{fn}: L={L} blocks={nb} total {(dn[-1].max() - t0) / 1e3:.1f} us")
    print(f"{'lvl':>4} {'span us':>8} {'busy med':>9} {'busy max':>9} {'tail us':>8}")
    tot_busy = tot_tail = 0
    for k in range(L):
        nxt = st[k + 1].min() if k + 1 < L else dn[k].max()
        span = nxt - st[k].min()
        busy = dn[k] - st[k]
        tail = nxt - dn[k].max()
        tot_busy += busy.max()
        tot_tail += max(0, tail)
        print(f"{k:4d} {span / 1e3:8.2f} {np.median(busy) / 1e3:9.2f} {busy.max() / 1e3:9.2f} "
              f"{tail / 1e3:8.2f}")
    print(f"sum of max busy {tot_busy / 1e3:.1f} us, sum of barrier tails {tot_tail / 1e3:.1f} us")


if __name__ == "__main__":
    for f in sys.argv[1:]:
        main(f)
