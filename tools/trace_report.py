"""Analyse an HF_TRACE dump: per-level critical path composition.

record = {level, cta, t_top, t_ready, t_computed, t_published, edges, rows} (ns)
For the LAST-published piece of every level: wait = ready - previous level done,
split into 'own' (its CTA still busy: staging / previous piece) and 'wake'.
"""
import sys

import numpy as np


def main(fn):
    a = np.fromfile(fn, dtype=np.uint64).reshape(-1, 8).astype(np.int64)
    lv, cta, ttop, trdy, tcmp, tpub, E, nn = a.T
    fwd = "_fwd" in fn
    levels = np.unique(lv)
    order = levels if fwd else levels[::-1]
    done = {k: tpub[lv == k].max() for k in order}
    # previous piece end per CTA
    idx = np.lexsort((ttop, cta))
    prev_end = np.full(len(a), -1, np.int64)
    for i0, i1 in zip(idx[:-1], idx[1:]):
        if cta[i0] == cta[i1]:
            prev_end[i1] = tpub[i0]
    rec = []
    prev = None
    for k in order:
        sel = np.nonzero(lv == k)[0]
        last = sel[np.argmax(tpub[sel])]
        if prev is not None:
            d0 = done[prev]
            rec.append((done[k] - d0, trdy[last] - d0, ttop[last] - d0, tcmp[last] - trdy[last],
                        tpub[last] - tcmp[last], E[last], nn[last], len(sel)))
        prev = k
    r = np.array(rec, dtype=np.float64)
    span = max(done.values()) - ttop.min()
    print(f"{fn.split('/')[-1]}: {len(a)} pieces, {len(levels)} levels, {span / 1e3:.0f} us, "
          f"{span / 1e3 / len(levels):.2f} us/level")
    names = ["gap", "ready-prevdone", "top-prevdone", "compute", "publish"]
    for i, nm in enumerate(names):
        print(f"   last piece {nm:15s} median {np.median(r[:, i]) / 1e3:6.2f} us  "
              f"p90 {np.percentile(r[:, i], 90) / 1e3:6.2f}")
    print(f"   last piece edges median {np.median(r[:, 5]):.0f} max {r[:, 5].max():.0f}; "
          f"all pieces edges median {np.median(E):.0f} max {E.max()}; pieces/level {np.median(r[:, 7]):.0f}")
    dc = tcmp - trdy
    print(f"   compute all pieces median {np.median(dc) / 1e3:.2f} us p90 {np.percentile(dc, 90) / 1e3:.2f} "
          f"max {dc.max() / 1e3:.2f}; heavy (E>ecap?) count {(E > np.median(E) * 1.8).sum()}")


if __name__ == "__main__":
    for f in sys.argv[1:]:
        main(f)
