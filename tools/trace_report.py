"""Analyse an HF_TRACE dump of the dataflow propagation kernel.

File: int32 header {ntask, L, S, SC}, int32 tb[L+1] (first task of pass-level q),
then per task uint64 {warp, t_start, t_ready0, t_ready_all, t_done, info, 0, 0}
(globaltimer ns): t_ready0 = first gather batch final, t_ready_all = every gather
batch final and the staged delays landed, t_done = the task's stores issued;
info = poll rounds << 32 | edges << 16 | rows.

Per pass-level q: done_q = last t_done of the level.  The task that finishes last
is the level's critical task; its time after done_{q-1} splits into: late start
(its warp was still busy with an earlier task), wait (first gather batch: inputs
not yet visible + gather latency), more batches (further gather batches and the
delay copies) and compute+store (ready_all -> done).
"""
import sys

import numpy as np


def main(fn):
    raw = np.fromfile(fn, dtype=np.int32)
    ntask, L, S, SC = (int(x) for x in raw[:4])
    tb = raw[4:4 + L + 1].astype(np.int64)
    off = (4 + L + 1) * 4
    a = np.frombuffer(open(fn, "rb").read()[off:], dtype=np.uint64).reshape(-1, 8).astype(np.int64)
    a = a[:ntask]
    w, ts, tr0, tra, td, info = a[:, 0], a[:, 1], a[:, 2], a[:, 3], a[:, 4], a[:, 5]
    npoll, E, NR = info >> 32, (info >> 16) & 0xffff, info & 0xffff
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
    rows = {k: [] for k in ("late start", "wait (batch 0)", "more batches + delays",
                            "compute+store", "poll rounds", "edges", "rows")}
    for q in range(1, L):
        sel = np.arange(tb[q], tb[q + 1])
        if len(sel) == 0:
            continue
        i = sel[np.argmax(td[sel])]
        base = done[q - 1]
        rows["late start"].append(max(0, ts[i] - base))
        rows["wait (batch 0)"].append(tr0[i] - max(ts[i], base))
        rows["more batches + delays"].append(tra[i] - tr0[i])
        rows["compute+store"].append(td[i] - tra[i])
        rows["poll rounds"].append(npoll[i] * 1000)
        rows["edges"].append(E[i] * 1000)
        rows["rows"].append(NR[i] * 1000)
    dur = td - ts
    print(f"{fn}: {ntask} tasks, {L} levels, S={S} SC={SC}, {span / 1e3:.1f} us, "
          f"{span / 1e3 / L:.2f} us/level, warps {len(np.unique(w))}")
    print(f"   level gap                     median {np.median(gaps) / 1e3:6.2f} us  "
          f"p90 {np.percentile(gaps, 90) / 1e3:6.2f}")
    for nm, v in rows.items():
        v = np.array(v) / 1e3
        unit = "us" if nm not in ("poll rounds", "edges", "rows") else "  "
        print(f"   critical task {nm:22s} median {np.median(v):6.2f} {unit}  "
              f"p90 {np.percentile(v, 90):6.2f}  mean {v.mean():6.2f}")
    print(f"   all tasks: start->ready0 median {np.median(tr0 - ts) / 1e3:.2f} us, "
          f"ready0->ready_all {np.median(tra - tr0) / 1e3:.2f} us, ready_all->done "
          f"{np.median(td - tra) / 1e3:.2f} us, duration p90 {np.percentile(dur, 90) / 1e3:.2f} us; "
          f"poll rounds mean {npoll.mean():.2f}, tasks with >=1 poll {np.mean(npoll > 0):.2f}; "
          f"edges mean {E.mean():.1f}, rows mean {NR.mean():.1f}")
    ahead = ts - np.where(lvl > 0, done[np.maximum(lvl - 1, 0)], t0)
    print(f"   task start - pred level done: median {np.median(ahead) / 1e3:.2f} us "
          f"(negative = started before its inputs were complete)")


if __name__ == "__main__":
    for f in sys.argv[1:]:
        main(f)
