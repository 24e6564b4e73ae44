"""Analyse an HF_TRACE dump of the dataflow propagation kernel.

File: int32 header {ntask, L, S, SC}, int32 tb[L+1] (first task of pass-level q),
then per task uint64 {warp, t_start, t_ready, t_done} (globaltimer ns;
t_ready = first gather batch complete, i.e. its inputs were final).

Per pass-level q: done_q = last t_done of the level.  For the task that finishes
last, split its time after done_{q-1} into: late start (its warp was still busy
with an earlier task), wait (inputs not yet visible / gather latency) and
compute+store (ready -> done).
"""
import sys

import numpy as np


def main(fn):
    raw = np.fromfile(fn, dtype=np.int32)
    ntask, L, S, SC = (int(x) for x in raw[:4])
    tb = raw[4:4 + L + 1].astype(np.int64)
    off = (4 + L + 1) * 4
    a = np.frombuffer(open(fn, "rb").read()[off:], dtype=np.uint64).reshape(-1, 4).astype(np.int64)
    a = a[:ntask]
    w, ts, tr, td = a.T
    ok = td > 0
    t0 = ts[ok].min()
    span = td[ok].max() - t0
    lvl = np.searchsorted(tb, np.arange(ntask), side="right") - 1
    done = np.zeros(L, np.int64)
    for q in range(L):
        sel = np.arange(tb[q], tb[q + 1])
        sel = sel[ok[sel]]
        done[q] = td[sel].max() if len(sel) else (done[q - 1] if q else t0)
    gaps = np.diff(np.concatenate([[t0], done]))
    late, wait, comp = [], [], []
    for q in range(1, L):
        sel = np.arange(tb[q], tb[q + 1])
        if len(sel) == 0:
            continue
        i = sel[np.argmax(td[sel])]
        base = done[q - 1]
        late.append(max(0, ts[i] - base))
        wait.append(tr[i] - max(ts[i], base))
        comp.append(td[i] - tr[i])
    dur = td - ts
    print(f"{fn}: {ntask} tasks, {L} levels, S={S} SC={SC}, {span / 1e3:.1f} us, "
          f"{span / 1e3 / L:.2f} us/level")
    print(f"   level gap        median {np.median(gaps) / 1e3:6.2f} us  p90 {np.percentile(gaps, 90) / 1e3:6.2f}")
    for nm, v in (("last task late start", late), ("last task wait", wait),
                  ("last task compute+store", comp)):
        v = np.array(v) / 1e3
        print(f"   {nm:24s} median {np.median(v):6.2f} us  p90 {np.percentile(v, 90):6.2f}")
    print(f"   all tasks: start->ready median {np.median(tr - ts) / 1e3:.2f} us, "
          f"ready->done median {np.median(td - tr) / 1e3:.2f} us, duration p90 "
          f"{np.percentile(dur, 90) / 1e3:.2f} us; warps {len(np.unique(w))}")
    # how far ahead of the front do warps start their tasks?
    q_of = lvl
    ahead = ts - np.where(q_of > 0, done[np.maximum(q_of - 1, 0)], t0)
    print(f"   task start - pred level done: median {np.median(ahead) / 1e3:.2f} us "
          f"(negative = started before its inputs were complete)")


if __name__ == "__main__":
    for f in sys.argv[1:]:
        main(f)
