"""CPU oracle for the DAG-propagation hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2203_08395_b200``) never imports, links or executes it, and the two
share no code: the oracle is ``oracle.c`` (plain sequential C, see its header
for the PAPER.md / BASELINE.json passages each function follows), compiled with
gcc (``-O2 -fno-fast-math -ffp-contract=off``) into ``liboracle.so`` and called
here through ctypes.  This wrapper is argument marshalling only.

Pins that tie the oracle to something other than itself live in
``tests/test_oracle_pins.py`` (Fig. 1 / Fig. 5 worked graphs, closed forms,
generator-known levels, brute-force path enumeration, exact-integer DFS,
invariants, metamorphic relations).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-std=c11", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared",
          "-pthread"]

OK, INVALID, BAD_CSR, CYCLE = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (in-tree)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32 = ctypes.c_int32
        lib.oracle_check_csr.argtypes = [i32, i32, P, P]
        lib.oracle_fanout.argtypes = [i32, i32, P, P, P, P, P]
        lib.oracle_check_fanout.argtypes = [i32, i32, P, P, P, P]
        lib.oracle_levelize.argtypes = [i32, i32, P, P, P, P, P, P, P, P, P]
        lib.oracle_forward.argtypes = [i32, i32, P, P, P, P, P, P]
        lib.oracle_forward_mode.argtypes = [i32, i32, P, P, P, P, P, P, ctypes.c_int]
        lib.oracle_backward_mode.argtypes = [i32, i32, P, P, P, ctypes.c_float, P, P, P, P, P,
                                             ctypes.c_int]
        lib.oracle_batch_mode.argtypes = [i32, i32, P, P, i32, P, ctypes.c_int, P, P, P, P, P,
                                          ctypes.c_int, ctypes.c_int]
        lib.oracle_backward.argtypes = [i32, i32, P, P, P, ctypes.c_float, P, P, P, P, P]
        lib.oracle_batch.argtypes = [i32, i32, P, P, i32, P, ctypes.c_int, P, P, P, P, P,
                                     ctypes.c_int]
        lib.oracle_critical_path.argtypes = [i32, i32, P, P, P, ctypes.c_int64, P,
                                             ctypes.c_float, P, i32, P]
        lib.oracle_critical_paths.argtypes = [i32, i32, P, P, i32, P, P, P, P, i32, P]
        lib.oracle_critical_paths_k.argtypes = [i32, i32, P, P, i32, P, P, P, i32, P, P, i32, P]
        lib.oracle_mis.argtypes = [i32, i32, P, P, P, P]
        for f in (lib.oracle_critical_paths_k, lib.oracle_mis, lib.oracle_check_csr, lib.oracle_check_fanout, lib.oracle_levelize,
                  lib.oracle_forward, lib.oracle_backward, lib.oracle_batch,
                  lib.oracle_critical_path, lib.oracle_critical_paths, lib.oracle_forward_mode,
                  lib.oracle_backward_mode, lib.oracle_batch_mode):
            f.restype = ctypes.c_int
        lib.oracle_fanout.restype = None
        _lib = lib
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


class OracleError(RuntimeError):
    def __init__(self, code: int, unready: int = 0):
        self.code = code
        self.unready = unready
        super().__init__({INVALID: "invalid argument", BAD_CSR: "bad CSR",
                          CYCLE: f"cycle ({unready} nodes never ready)"}.get(code, str(code)))


@dataclass
class Levels:
    level: np.ndarray        # int32 [n]
    level_ptr: np.ndarray    # int32 [L+1]
    order: np.ndarray        # int32 [n]
    topo: np.ndarray         # int32 [n]  (FIFO Kahn order; internal to the oracle)
    num_levels: int


def fanout(n, m, in_ptr, in_src):
    """Derived fan-out CSR (out_ptr, out_dst, out_eid): stable counting sort by source."""
    lib = _load()
    in_ptr, in_src = _i32(in_ptr), _i32(in_src)
    op = np.zeros(n + 1, np.int32)
    od = np.zeros(max(m, 1), np.int32)
    oe = np.zeros(max(m, 1), np.int32)
    lib.oracle_fanout(n, m, _p(in_ptr), _p(in_src), _p(op), _p(od), _p(oe))
    return op, od[:m], oe[:m]


def check_csr(n, m, in_ptr, in_src) -> int:
    return _load().oracle_check_csr(n, m, _p(_i32(in_ptr)), _p(_i32(in_src)))


def check_fanout(n, m, in_ptr, in_src, out_ptr, out_dst) -> int:
    return _load().oracle_check_fanout(n, m, _p(_i32(in_ptr)), _p(_i32(in_src)),
                                       _p(_i32(out_ptr)), _p(_i32(out_dst)))


def levelize(n, m, in_ptr, in_src) -> Levels:
    """FIFO Kahn levelization; raises OracleError(CYCLE, unready) on a cycle."""
    lib = _load()
    in_ptr, in_src = _i32(in_ptr), _i32(in_src)
    topo = np.zeros(max(n, 1), np.int32)
    level = np.zeros(max(n, 1), np.int32)
    lptr = np.zeros(n + 2, np.int32)
    order = np.zeros(max(n, 1), np.int32)
    nt, L, un = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
    rc = lib.oracle_levelize(n, m, _p(in_ptr), _p(in_src), _p(topo), ctypes.byref(nt),
                             _p(level), _p(lptr), _p(order), ctypes.byref(L),
                             ctypes.byref(un))
    if rc:
        raise OracleError(rc, un.value)
    return Levels(level[:n].copy(), lptr[:L.value + 1].copy(), order[:n].copy(),
                  topo[:n].copy(), L.value)


def forward(n, m, in_ptr, in_src, delay, at_src=None, lv: Optional[Levels] = None,
            early: bool = False):
    """at[n] = max-plus arrival times (at_src None => +0 at sources; delay None => +0);
    early=True: min-plus (hold-analysis arrival, NEXT-2, reading R18)."""
    lib = _load()
    in_ptr, in_src = _i32(in_ptr), _i32(in_src)
    lv = lv or levelize(n, m, in_ptr, in_src)
    d = None if delay is None else _f32(delay)
    a = None if at_src is None else _f32(at_src)
    at = np.zeros(max(n, 1), np.float32)
    rc = lib.oracle_forward_mode(n, m, _p(in_ptr), _p(in_src), _p(d), _p(a), _p(lv.topo),
                                 _p(at), int(early))
    if rc:
        raise OracleError(rc)
    return at[:n]


def backward(n, m, in_ptr, in_src, delay, t_req, at, lv: Optional[Levels] = None,
             early: bool = False):
    """(rat[n], slack[n], wns) by min-plus over fan-out; T at every sink.
    early=True: max-plus, slack = at - rat (hold mode, NEXT-2, reading R18)."""
    lib = _load()
    in_ptr, in_src = _i32(in_ptr), _i32(in_src)
    lv = lv or levelize(n, m, in_ptr, in_src)
    d = None if delay is None else _f32(delay)
    at = _f32(at)
    rat = np.zeros(max(n, 1), np.float32)
    slack = np.zeros(max(n, 1), np.float32)
    wns = ctypes.c_float(0.0)
    rc = lib.oracle_backward_mode(n, m, _p(in_ptr), _p(in_src), _p(d), ctypes.c_float(t_req),
                                  _p(lv.topo), _p(at), _p(rat), _p(slack), ctypes.byref(wns),
                                  int(early))
    if rc:
        raise OracleError(rc)
    return rat[:n], slack[:n], np.float32(wns.value)


def batch(n, m, in_ptr, in_src, delays, t_req, at_src=None, layout: str = "ms",
          threads: int = 1, want_at_rat: bool = False, early: bool = False):
    """S scenarios: delays [m][S] ("ms") or [S][m] ("sm"); t_req[S].
    Returns wns[S] (and at[n][S], rat[n][S] if want_at_rat)."""
    lib = _load()
    in_ptr, in_src = _i32(in_ptr), _i32(in_src)
    delays = _f32(delays)
    S = delays.shape[1] if layout == "ms" else delays.shape[0]
    t = _f32(np.broadcast_to(np.asarray(t_req, np.float32), (S,)))
    a = None if at_src is None else _f32(at_src)
    wns = np.zeros(max(S, 1), np.float32)
    at_all = np.zeros((n, S), np.float32) if want_at_rat else None
    rat_all = np.zeros((n, S), np.float32) if want_at_rat else None
    rc = lib.oracle_batch_mode(n, m, _p(in_ptr), _p(in_src), S, _p(delays),
                               0 if layout == "sm" else 1, _p(t), _p(a), _p(wns), _p(at_all),
                               _p(rat_all), threads, int(early))
    if rc:
        raise OracleError(rc)
    if want_at_rat:
        return wns[:S], at_all, rat_all
    return wns[:S]


def critical_path(n, m, in_ptr, in_src, delay, at, t_req, max_len=None):
    """NEXT-1 (reading R17): nodes of the critical path of the worst endpoint,
    endpoint first, source last (one delay set in fan-in edge order)."""
    lib = _load()
    in_ptr, in_src = _i32(in_ptr), _i32(in_src)
    d = _f32(delay) if m else np.zeros(1, np.float32)
    at = _f32(at) if n else np.zeros(1, np.float32)
    max_len = max(1, n if max_len is None else max_len)
    path = np.zeros(max_len, np.int32)
    ln = ctypes.c_int32(0)
    rc = lib.oracle_critical_path(n, m, _p(in_ptr), _p(in_src), _p(d), ctypes.c_int64(1), _p(at),
                                  ctypes.c_float(t_req), _p(path), max_len, ctypes.byref(ln))
    if rc:
        raise OracleError(rc)
    return path[:ln.value].copy()


def critical_paths(n, m, in_ptr, in_src, delays_ms, at_all, t_req, max_len=None):
    """S scenarios: delays [m][S], at [n][S], t_req[S] -> list of S paths."""
    lib = _load()
    in_ptr, in_src = _i32(in_ptr), _i32(in_src)
    delays_ms = _f32(delays_ms)
    S = delays_ms.shape[1]
    at_all = _f32(at_all)
    t = _f32(np.broadcast_to(np.asarray(t_req, np.float32), (S,)))
    max_len = max(1, n if max_len is None else max_len)
    paths = np.zeros((S, max_len), np.int32)
    lens = np.zeros(S, np.int32)
    rc = lib.oracle_critical_paths(n, m, _p(in_ptr), _p(in_src), S, _p(delays_ms), _p(at_all),
                                   _p(t), _p(paths), max_len, _p(lens))
    if rc:
        raise OracleError(rc)
    return [paths[s, :lens[s]].copy() for s in range(S)]


def critical_paths_k(n, m, in_ptr, in_src, delays_ms, at_all, t_req, K, max_len=None):
    """Top-K endpoints per scenario (NEXT-1, reading R17): delays [m][S], at [n][S],
    t_req[S] -> (endpoints [S][K], list over s of K paths); endpoint -1 / empty path
    past the number of sinks."""
    lib = _load()
    in_ptr, in_src = _i32(in_ptr), _i32(in_src)
    delays_ms = _f32(delays_ms)
    S = delays_ms.shape[1]
    at_all = _f32(at_all)
    t = _f32(np.broadcast_to(np.asarray(t_req, np.float32), (S,)))
    max_len = max(1, n if max_len is None else max_len)
    ends = np.zeros((S, K), np.int32)
    paths = np.zeros((S, K, max_len), np.int32)
    lens = np.zeros((S, K), np.int32)
    rc = lib.oracle_critical_paths_k(n, m, _p(in_ptr), _p(in_src), S, _p(delays_ms), _p(at_all),
                                     _p(t), K, _p(ends), _p(paths), max_len, _p(lens))
    if rc:
        raise OracleError(rc)
    return ends, [[paths[s, r, :lens[s, r]].copy() for r in range(K)] for s in range(S)]


def mis(n, m, in_ptr, in_src, prio):
    """NEXT-4 (reading R19): lexicographically-first maximal independent set of the
    undirected graph of the edges, vertices visited by increasing (prio, id).
    Returns uint8 in_set[n]."""
    lib = _load()
    in_ptr, in_src = _i32(in_ptr), _i32(in_src)
    pr = _i32(prio) if n else np.zeros(1, np.int32)
    out = np.zeros(max(n, 1), np.uint8)
    rc = lib.oracle_mis(n, m, _p(in_ptr), _p(in_src), _p(pr), _p(out))
    if rc:
        raise OracleError(rc)
    return out[:n].copy()
