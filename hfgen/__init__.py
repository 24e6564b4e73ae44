"""Seeded synthetic inputs for the DAG-propagation hot path.

This module is the ONE thing the CPU oracle (``oracle/``) and the CUDA path
(``paper_2203_08395_b200``) share: it produces graphs (CSR fan-in), per-edge
fp32 delays, source arrival times and what-if scenario delays.  It holds none
of the method's arithmetic (no levelization, no max-plus / min-plus); the
levels it returns for the levelized generator are the generator's own labels
(pin P5), known by construction.

Randomness is counter based: every draw is ``splitmix64`` of
(seed, stream, index), so any slice of any array (e.g. one rank's block of
scenarios) can be regenerated independently and bit-identically.
``u = (h >> 40) * 2**-24`` is a 24-bit uniform in [0, 1).

Configs (BASELINE.json:7-11, recipe in SURVEY.md §8(d) and DESIGN.md §3):
  C1  levelized circuit DAG, n=10k, m=20k, D=50, seed 1
  C2  chain / binary out-tree / random in-degree-2 DAG, n=1M, seed 2
  C3  levelized circuit DAG, n=1.5M, m=2.5M, D=200, seed 3
  C4  the C3 graph (seed 4) with S=64 scenario delay sets
  C5  power-law fan-in DAG, n=10M, max in-degree 10k, seed 5
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import os

import numpy as np

__all__ = [
    "Graph", "splitmix64", "hash3", "uniform", "levelized", "chain", "bintree",
    "random_dag", "powerlaw", "scenario_delays", "config", "CONFIGS",
]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)

# stream ids (fixed forever: changing one changes every generated input)
S_LEVEL_PERM = 1
S_EXTRA = 16          # + attempt (resampling rounds)
S_IDS = 2
S_DELAY = 3
S_ATSRC = 4
S_CHAIN = 5
S_RAND_A = 6
S_RAND_B = 7
S_PL_K = 8
S_PL_PRED = 64        # + attempt
S_SCEN = 1 << 20      # + scenario index


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def hash3(seed: int, stream: int, index) -> np.ndarray:
    """64-bit hash of (seed, stream, index); index may be an array."""
    base = splitmix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    with np.errstate(over="ignore"):
        base = splitmix64(base ^ np.uint64(stream & 0xFFFFFFFFFFFFFFFF))
        idx = np.asarray(index, dtype=np.uint64)
        return splitmix64(base + idx * _GAMMA)


def uniform(seed: int, stream: int, index) -> np.ndarray:
    """24-bit uniform in [0,1) as float64: (h >> 40) * 2^-24."""
    h = hash3(seed, stream, index)
    return (h >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)


@dataclasses.dataclass
class Graph:
    """A DAG as CSR fan-in (rows = sink node id), plus generator metadata."""
    name: str
    n: int
    m: int
    in_ptr: np.ndarray            # int32 [n+1]
    in_src: np.ndarray            # int32 [m]
    delay: np.ndarray             # float32 [m], indexed by fan-in position
    at_src: np.ndarray            # float32 [n] (only in-degree-0 entries matter)
    t_req: float                  # required time T at every sink
    seed: int
    level_label: Optional[np.ndarray] = None   # int32 [n], generator-known level
    depth: Optional[int] = None

    def edges(self):
        """(src, dst) int64 arrays in fan-in order."""
        dst = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.in_ptr))
        return self.in_src.astype(np.int64), dst


def _delays(seed: int, m: int) -> np.ndarray:
    # d = float32(5.0 + 45.0*u) computed in float64 and rounded once (§8(d))
    return (5.0 + 45.0 * uniform(seed, S_DELAY, np.arange(m))).astype(np.float32)


def _at_src(seed: int, n: int) -> np.ndarray:
    return (20.0 * uniform(seed, S_ATSRC, np.arange(n))).astype(np.float32)


def _id_perm(seed: int, n: int, relabel: bool) -> np.ndarray:
    """id_of_position[p]: a seeded random permutation (ids carry no order)."""
    if not relabel:
        return np.arange(n, dtype=np.int64)
    key = hash3(seed, S_IDS, np.arange(n))
    order = np.argsort(key, kind="stable")
    ids = np.empty(n, dtype=np.int64)
    ids[order] = np.arange(n, dtype=np.int64)
    return ids


def _build(name, n, src_pos, dst_pos, ids, seed, t_req, level_pos=None, depth=None,
           delays=True) -> Graph:
    """Relabel positions to ids and build CSR fan-in; rows keep generation order."""
    src = ids[src_pos] if len(src_pos) else np.zeros(0, np.int64)
    dst = ids[dst_pos] if len(dst_pos) else np.zeros(0, np.int64)
    order = np.argsort(dst, kind="stable")
    src = src[order]
    dst = dst[order]
    m = int(len(src))
    counts = np.bincount(dst, minlength=n) if m else np.zeros(n, np.int64)
    in_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=in_ptr[1:])
    lab = None
    if level_pos is not None:
        lab = np.empty(n, dtype=np.int32)
        lab[ids] = level_pos
    return Graph(name=name, n=n, m=m, in_ptr=in_ptr.astype(np.int32),
                 in_src=src.astype(np.int32),
                 delay=_delays(seed, m) if delays else np.zeros(m, np.float32),
                 at_src=_at_src(seed, n), t_req=float(t_req), seed=seed,
                 level_label=lab, depth=depth)


def levelized(n: int, m: int, depth: int, seed: int, relabel: bool = True,
              endpoint_frac: float = 0.04, window: int = 8, name: str = "levelized") -> Graph:
    """Levelized "circuit-shaped" DAG (used by C1, C3, C4).

    Position p sits at level floor(p*D/n).  Every node of level l>=1 gets one
    anchor predecessor in level l-1 (drawn from the 96% of l-1 that are not
    endpoints), and R = m - (n - |level 0|) extra edges attach to uniform
    non-source nodes from a level in [l-8, l-1] with a u^3-skewed index
    (heavy-tailed fan-out).  Duplicate (u,v) pairs are redrawn.  So the level
    of every node is its generator label (pin P5).
    """
    if depth < 1 or n < depth:
        raise ValueError("need 1 <= depth <= n")
    pos = np.arange(n, dtype=np.int64)
    lvl = (pos * depth) // n
    sizes = np.bincount(lvl, minlength=depth).astype(np.int64)
    lstart = np.zeros(depth + 1, dtype=np.int64)
    np.cumsum(sizes, out=lstart[1:])
    n_anchor = n - int(sizes[0])
    if m < n_anchor:
        raise ValueError(f"m={m} < anchor edges {n_anchor}")
    # per-level random permutation: sort positions by (level, key)
    key = hash3(seed, S_LEVEL_PERM, pos)
    perm = np.lexsort((key, lvl))                      # positions, grouped by level
    csize = np.maximum(1, np.floor(sizes * (1.0 - endpoint_frac)).astype(np.int64))
    # anchors: j-th node of level l -> C_{l-1}[j mod |C_{l-1}|]
    v_a = pos[lstart[1]:]
    l_a = lvl[lstart[1]:]
    j = v_a - lstart[l_a]
    u_a = perm[lstart[l_a - 1] + (j % csize[l_a - 1])]
    # extra edges, with resampling of duplicates
    R = m - n_anchor
    nonsrc = n - int(lstart[1])
    if R > 0 and nonsrc == 0:
        raise ValueError("extra edges need a non-source level")
    ridx = np.arange(R, dtype=np.int64)
    ev = np.empty(R, np.int64)
    eu = np.empty(R, np.int64)

    def draw(idx, attempt):
        st = S_EXTRA + attempt
        u1 = uniform(seed, st, 3 * idx)
        u2 = uniform(seed, st, 3 * idx + 1)
        u3 = uniform(seed, st, 3 * idx + 2)
        v = lstart[1] + np.floor(u1 * nonsrc).astype(np.int64)
        lv = lvl[v]
        lo = np.maximum(0, lv - window)
        lp = lo + np.floor(u2 * (lv - lo)).astype(np.int64)
        k = np.floor(sizes[lp] * u3 ** 3).astype(np.int64)
        return lstart[lp] + k, v

    todo = ridx
    attempt = 0
    base_keys = v_a * n + u_a                      # anchors are never resampled
    while len(todo):
        eu[todo], ev[todo] = draw(todo, attempt)
        keys = np.concatenate([base_keys, ev * n + eu])
        order = np.argsort(keys, kind="stable")    # anchors first, then extras by index
        sk = keys[order]
        dup = np.zeros(len(keys), dtype=bool)
        dup[order[1:]] = sk[1:] == sk[:-1]
        todo = np.nonzero(dup[n_anchor:])[0].astype(np.int64)
        attempt += 1
        if attempt > 64:
            raise RuntimeError("duplicate resampling did not converge")
    src_pos = np.concatenate([u_a, eu])
    dst_pos = np.concatenate([v_a, ev])
    ids = _id_perm(seed, n, relabel)
    t_req = 0.9 * 27.5 * (depth - 1)
    return _build(name, n, src_pos, dst_pos, ids, seed, t_req, level_pos=lvl, depth=depth)


def chain(n: int, seed: int = 2, relabel: bool = True) -> Graph:
    """Linear chain k -> k+1 (C2)."""
    p = np.arange(max(n - 1, 0), dtype=np.int64)
    ids = _id_perm(seed, n, relabel)
    return _build("chain", n, p, p + 1, ids, seed, t_req=0.0,
                  level_pos=np.arange(n, dtype=np.int64), depth=n)


def bintree(n: int, seed: int = 2, relabel: bool = True) -> Graph:
    """Binary out-tree i -> 2i+1, 2i+2 (C2)."""
    c = np.arange(1, n, dtype=np.int64)
    parent = (c - 1) // 2
    ids = _id_perm(seed, n, relabel)
    x = np.arange(1, n + 1, dtype=np.int64)          # heap index + 1
    lv = np.floor(np.log2(x.astype(np.float64))).astype(np.int64)
    lv = np.where((np.int64(1) << (lv + 1)) <= x, lv + 1, lv)   # guard float log2
    lv = np.where((np.int64(1) << lv) > x, lv - 1, lv)
    return _build("bintree", n, parent, c, ids, seed, t_req=0.0, level_pos=lv,
                  depth=int(lv.max()) + 1 if n else 0)


def random_dag(n: int, seed: int = 2, relabel: bool = True) -> Graph:
    """Node 0 is the source, node 1 has pred 0, v>=2 has 2 distinct uniform preds in [0,v) (C2)."""
    v = np.arange(2, n, dtype=np.int64)
    p1 = np.floor(uniform(seed, S_RAND_A, v) * v).astype(np.int64)
    p2 = np.floor(uniform(seed, S_RAND_B, v) * (v - 1)).astype(np.int64)
    p2 = np.where(p2 >= p1, p2 + 1, p2)
    src = np.concatenate([np.zeros(1 if n >= 2 else 0, np.int64),
                          np.stack([p1, p2], 1).reshape(-1)])
    dst = np.concatenate([np.ones(1 if n >= 2 else 0, np.int64), np.repeat(v, 2)])
    ids = _id_perm(seed, n, relabel)
    return _build("random_dag", n, src, dst, ids, seed, t_req=0.0)


def powerlaw(n: int, seed: int = 5, alpha: float = 2.5, kmax: int = 10_000,
             source_frac: float = 0.01, plant: bool = True, relabel: bool = True) -> Graph:
    """Power-law fan-in DAG (C5): first 1% sources; P(k) ~ k^-alpha on [1,kmax];
    distinct uniform preds in [0,v); the last position planted with exactly kmax preds.
    k is clamped to floor(v/2) so distinct sampling terminates (never binds at n=1e7)."""
    nsrc = max(1, int(n * source_frac))
    v = np.arange(nsrc, n, dtype=np.int64)
    ks = np.arange(1, kmax + 1, dtype=np.float64)
    pmf = ks ** (-alpha)
    cdf = np.cumsum(pmf) / pmf.sum()
    u = uniform(seed, S_PL_K, v)
    k = np.searchsorted(cdf, u, side="right").astype(np.int64) + 1
    k = np.minimum(k, kmax)
    if plant and len(v):
        k[-1] = kmax
    k = np.minimum(k, v // 2)
    k = np.maximum(k, np.minimum(1, v))
    rowptr = np.zeros(len(v) + 1, np.int64)
    np.cumsum(k, out=rowptr[1:])
    M = int(rowptr[-1])
    row = np.repeat(np.arange(len(v), dtype=np.int64), k)
    dstv = v[row]
    slot = np.arange(M, dtype=np.int64)
    pred = np.empty(M, np.int64)
    todo = slot
    attempt = 0
    while len(todo):
        uu = uniform(seed, S_PL_PRED + attempt, todo)
        pred[todo] = np.floor(uu * dstv[todo]).astype(np.int64)
        keys = dstv * n + pred
        order = np.argsort(keys, kind="stable")
        sk = keys[order]
        dup = np.zeros(M, dtype=bool)
        dup[order[1:]] = sk[1:] == sk[:-1]
        todo = np.nonzero(dup)[0].astype(np.int64)
        attempt += 1
        if attempt > 200:
            raise RuntimeError("pred resampling did not converge")
    ids = _id_perm(seed, n, relabel)
    return _build("powerlaw", n, pred, dstv, ids, seed, t_req=0.0)


def scenario_delays(g: Graph, s_begin: int, s_end: int, layout: str = "ms") -> np.ndarray:
    """What-if delay sets d_s[e] = float32(float64(d[e]) * (0.9 + 0.2*u_{s,e})) for
    global scenario ids s in [s_begin, s_end).  layout "ms" -> [m][S] (scenario-minor),
    "sm" -> [S][m]."""
    S = s_end - s_begin
    out = np.empty((S, g.m), dtype=np.float32)
    d64 = g.delay.astype(np.float64)
    idx = np.arange(g.m)

    def one(i):
        s = s_begin + i
        out[i] = (d64 * (0.9 + 0.2 * uniform(g.seed, S_SCEN + s, idx))).astype(np.float32)

    # rows are independent (keyed by global scenario id): numpy releases the GIL in
    # its ufuncs, so large sweeps (NEXT-3, S up to 1024) generate on all host cores
    if S * g.m >= (1 << 24):
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
            list(ex.map(one, range(S)))
    else:
        for i in range(S):
            one(i)
    if layout == "sm":
        return out
    if layout == "ms":
        return np.ascontiguousarray(out.T)
    raise ValueError(layout)


CONFIGS = {
    "C1": dict(kind="levelized", n=10_000, m=20_000, depth=50, seed=1),
    "C2-chain": dict(kind="chain", n=1_000_000, seed=2),
    "C2-tree": dict(kind="bintree", n=1_000_000, seed=2),
    "C2-random": dict(kind="random_dag", n=1_000_000, seed=2),
    "C3": dict(kind="levelized", n=1_500_000, m=2_500_000, depth=200, seed=3),
    "C4": dict(kind="levelized", n=1_500_000, m=2_500_000, depth=200, seed=4, scenarios=64),
    "C5": dict(kind="powerlaw", n=10_000_000, seed=5),
}


def config(name: str, scale: float = 1.0) -> Graph:
    """Build config `name`; `scale` < 1 shrinks n and m proportionally (parity-size runs)."""
    c = dict(CONFIGS[name])
    kind = c.pop("kind")
    c.pop("scenarios", None)
    if scale != 1.0:
        c["n"] = max(16, int(c["n"] * scale))
        if "m" in c:
            c["m"] = max(c["n"], int(c["m"] * scale))
        if "depth" in c:
            c["depth"] = max(2, min(c["depth"], c["n"] // 4))
    fn = {"levelized": levelized, "chain": chain, "bintree": bintree,
          "random_dag": random_dag, "powerlaw": powerlaw}[kind]
    if kind == "powerlaw" and scale != 1.0:
        c["kmax"] = max(2, min(10_000, c["n"] // 20))
    g = fn(**c)
    g.name = name
    return g
