"""Thin ctypes binding of libhf.so (include/hf.h).  Argument marshalling only:
every step of the path runs in the library's CUDA kernels.

Each ``hf_*`` function here has the name of the C entry point it calls.  Arrays
may be numpy arrays (host-pointer variant, synchronous) or CUDA torch tensors
(``_d`` variant on the graph's stream); the two cannot be mixed in one call.
There is no CPU fallback: if libhf.so is missing or fails to load, importing
this module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HF_LIB: an alternative in-tree build (A/B timing of kernel variants in tools/)
LIB_PATH = os.environ.get("HF_LIB") or os.path.join(_HERE, "libhf.so")

HF_OK, HF_ERR_INVALID_ARG, HF_ERR_BAD_CSR, HF_ERR_CYCLE = 0, 1, 2, 3
HF_ERR_NOT_LEVELIZED, HF_ERR_OOM, HF_ERR_CUDA, HF_ERR_NCCL = 4, 5, 6, 7
HF_LAYOUT_SM, HF_LAYOUT_MS = 0, 1

# every exported entry point of include/hf.h (checked by tests/test_abi.py)
EXPORTS = [
    "hf_last_error", "hf_status_string", "hf_version", "hf_graph_create", "hf_graph_create_d",
    "hf_graph_destroy", "hf_graph_set_stream", "hf_graph_info", "hf_sync", "hf_levelize",
    "hf_levelize_d", "hf_propagate_forward", "hf_propagate_forward_d", "hf_propagate_backward",
    "hf_propagate_backward_d", "hf_run_batch", "hf_run_batch_d", "hf_nccl_unique_id",
    "hf_nccl_comm_init", "hf_nccl_comm_destroy", "hf_profile_enable", "hf_profile_read",
    "hf_profile_read_batch", "hf_critical_path", "hf_critical_path_d", "hf_graph_set_mode",
    "hf_mis", "hf_mis_d", "hf_analyze", "hf_critical_paths_d",
]


class HFError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        super().__init__(f"{_status_name(status)}: {message}")


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -m paper_2203_08395_b200.build` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P, i32, i64, f32, c_int = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float,
                               ctypes.c_int)
    sig = {
        "hf_last_error": (ctypes.c_char_p, []),
        "hf_status_string": (ctypes.c_char_p, [c_int]),
        "hf_version": (c_int, []),
        "hf_graph_create": (c_int, [i32, i32, P, P, P, P, P, c_int, P, P]),
        "hf_graph_create_d": (c_int, [i32, i32, P, P, P, P, P, c_int, P, P]),
        "hf_graph_destroy": (c_int, [P]),
        "hf_graph_set_stream": (c_int, [P, P]),
        "hf_graph_set_mode": (c_int, [P, c_int]),
        "hf_mis": (c_int, [P, P, P]),
        "hf_mis_d": (c_int, [P, P, P]),
        "hf_graph_info": (c_int, [P, P, P, P]),
        "hf_sync": (c_int, [P]),
        "hf_levelize": (c_int, [P, P, P, P, P]),
        "hf_levelize_d": (c_int, [P, P, P, P, P]),
        "hf_propagate_forward": (c_int, [P, P, P]),
        "hf_propagate_forward_d": (c_int, [P, P, P]),
        "hf_propagate_backward": (c_int, [P, f32, P, P, P, P]),
        "hf_propagate_backward_d": (c_int, [P, f32, P, P, P, P]),
        "hf_run_batch": (c_int, [P, i32, P, c_int, P, P, P, P, P]),
        "hf_run_batch_d": (c_int, [P, i32, P, c_int, P, P, P, P, P, P, P]),
        "hf_nccl_unique_id": (c_int, [P]),
        "hf_nccl_comm_init": (c_int, [P, c_int, c_int, c_int, P]),
        "hf_nccl_comm_destroy": (c_int, [P]),
        "hf_profile_enable": (c_int, [P, c_int]),
        "hf_profile_read": (c_int, [P, P, P, P, P]),
        "hf_profile_read_batch": (c_int, [P, P]),
        "hf_critical_path_d": (c_int, [P, i32, P, P, P, f32, i32, P, P]),
        "hf_critical_path": (c_int, [P, P, f32, i32, P, P]),
        "hf_analyze": (c_int, [i32, i32, P, P, P, i32, P, P, P, P, P, c_int, P, P]),
        "hf_critical_paths_d": (c_int, [P, i32, P, P, P, f32, i32, i32, P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def _status_name(s: int) -> str:
    return _lib.hf_status_string(s).decode()


def _check(status: int):
    if status != HF_OK:
        raise HFError(status, _lib.hf_last_error().decode())


def _is_torch(x) -> bool:
    return x is not None and type(x).__module__.startswith("torch")


def _ptr(x):
    """Pointer of a numpy array / CUDA torch tensor (None -> NULL)."""
    if x is None:
        return None
    if _is_torch(x):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(x.data_ptr())
    if not x.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return x.ctypes.data_as(ctypes.c_void_p)


def _out(x, count: int, dtype, what: str):
    """A host output array: must be a C-contiguous `dtype` array of >= count elements
    (the library writes through its pointer; a wrong dtype or a short array would be
    garbled or overrun).  None passes through (optional outputs)."""
    if x is None or _is_torch(x):
        return x
    if not isinstance(x, np.ndarray) or x.dtype != np.dtype(dtype):
        raise TypeError(f"{what}: expected a numpy {np.dtype(dtype).name} array")
    if not x.flags["C_CONTIGUOUS"] or not x.flags["WRITEABLE"]:
        raise ValueError(f"{what}: array must be C-contiguous and writeable")
    if x.size < count:
        raise ValueError(f"{what}: needs >= {count} elements, has {x.size}")
    return x


def _np(x, dtype):
    return None if x is None else np.ascontiguousarray(x, dtype=dtype)


def _stream_of(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)   # torch.cuda.Stream


class Graph:
    """Owning handle of an hf_graph (destroyed with the object)."""

    def __init__(self, handle: ctypes.c_void_p, n: int, m: int, device: int):
        self._h = handle
        self.n, self.m, self.device = n, m, device

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            hf_graph_destroy(self)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def num_levels(self) -> int:
        return hf_graph_info(self)[2]


def hf_graph_create(n, m, fanin_ptr, fanin_src, fanout_ptr=None, fanout_dst=None, delay=None,
                    device: int = 0, stream=None) -> Graph:
    out = ctypes.c_void_p()
    if _is_torch(fanin_ptr):
        st = _lib.hf_graph_create_d(n, m, _ptr(fanin_ptr), _ptr(fanin_src), _ptr(fanout_ptr),
                                    _ptr(fanout_dst), _ptr(delay), device, _stream_of(stream),
                                    ctypes.byref(out))
    else:
        a = [_np(fanin_ptr, np.int32), _np(fanin_src, np.int32), _np(fanout_ptr, np.int32),
             _np(fanout_dst, np.int32), _np(delay, np.float32)]
        st = _lib.hf_graph_create(n, m, *[_ptr(x) for x in a], device, _stream_of(stream),
                                  ctypes.byref(out))
    _check(st)
    return Graph(out, n, m, device)


def hf_graph_destroy(g: Graph):
    _check(_lib.hf_graph_destroy(g.handle))


def hf_graph_set_stream(g: Graph, stream):
    _check(_lib.hf_graph_set_stream(g.handle, _stream_of(stream)))


def hf_graph_info(g: Graph):
    n, m, L = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(_lib.hf_graph_info(g.handle, ctypes.byref(n), ctypes.byref(m), ctypes.byref(L)))
    return n.value, m.value, L.value


def hf_sync(g: Graph):
    _check(_lib.hf_sync(g.handle))


def hf_levelize(g: Graph, level=None, level_ptr=None, order=None) -> int:
    """Levelize; optional outputs are filled in place (numpy => host variant,
    torch CUDA => device variant).  Returns L."""
    L = ctypes.c_int32()
    for x, what in ((level, "level"), (order, "order")):
        _out(x, g.n, np.int32, what)
    _out(level_ptr, 1, np.int32, "level_ptr")
    if level_ptr is not None and not _is_torch(level_ptr) and level_ptr.size < g.n + 1:
        raise ValueError("level_ptr: needs n + 1 elements")
    if any(_is_torch(x) for x in (level, level_ptr, order)):
        _check(_lib.hf_levelize_d(g.handle, ctypes.byref(L), _ptr(level), _ptr(level_ptr),
                                  _ptr(order)))
    else:
        _check(_lib.hf_levelize(g.handle, ctypes.byref(L), _ptr(level), _ptr(level_ptr),
                                _ptr(order)))
    return L.value


def levelize_np(g: Graph):
    """Convenience: (L, level, level_ptr, order) as numpy arrays."""
    level = np.zeros(max(g.n, 1), np.int32)
    lptr = np.zeros(g.n + 1, np.int32)
    order = np.zeros(max(g.n, 1), np.int32)
    L = hf_levelize(g, level, lptr, order)
    return L, level[:g.n], lptr[:L + 1], order[:g.n]


def hf_propagate_forward(g: Graph, at_src, at):
    if _is_torch(at):
        _check(_lib.hf_propagate_forward_d(g.handle, _ptr(at_src), _ptr(at)))
    else:
        _out(at, g.n, np.float32, "at")
        a = _np(at_src, np.float32)
        _check(_lib.hf_propagate_forward(g.handle, _ptr(a), _ptr(at)))


def hf_propagate_backward(g: Graph, t_req: float, at, rat, slack=None, wns=None):
    """wns: 1-element output (numpy float32 array or CUDA tensor) or None."""
    if _is_torch(rat):
        _check(_lib.hf_propagate_backward_d(g.handle, ctypes.c_float(t_req), _ptr(at), _ptr(rat),
                                            _ptr(slack), _ptr(wns)))
    else:
        _out(rat, g.n, np.float32, "rat")
        _out(slack, g.n, np.float32, "slack")
        _out(wns, 1, np.float32, "wns")
        a = _np(at, np.float32)
        _check(_lib.hf_propagate_backward(g.handle, ctypes.c_float(t_req), _ptr(a), _ptr(rat),
                                          _ptr(slack), _ptr(wns)))


HF_MODE_LATE, HF_MODE_EARLY = 0, 1


def hf_graph_set_mode(g: Graph, mode: int):
    """HF_MODE_LATE (setup, default) or HF_MODE_EARLY (hold) for later propagation calls."""
    _check(_lib.hf_graph_set_mode(g.handle, mode))


def hf_critical_path(g: Graph, at, t_req, max_len: int, path=None, path_len=None,
                     delays=None, s: int = 1):
    """NEXT-1 critical path of the worst endpoint (reading R17).

    Host: at (numpy [n]) with the graph's delays -> numpy array of node ids (endpoint
    first).  Device: at [n][S] CUDA tensor, delays [m][S] tensor (or None for the graph's
    delays, s == 1), t_req [S] tensor or float, path [S][max_len] and path_len [S] int32
    tensors (stream-ordered; path_len -1 marks an inconsistent at)."""
    if _is_torch(at):
        tr = t_req if _is_torch(t_req) else None
        ts = 0.0 if _is_torch(t_req) else float(t_req)
        _check(_lib.hf_critical_path_d(g.handle, s, _ptr(delays), _ptr(at), _ptr(tr),
                                       ctypes.c_float(ts), max_len, _ptr(path), _ptr(path_len)))
        return path, path_len
    a = _np(at, np.float32)
    out = np.zeros(max(1, max_len), np.int32)
    ln = ctypes.c_int32(0)
    _check(_lib.hf_critical_path(g.handle, _ptr(a), ctypes.c_float(t_req), max_len, _ptr(out),
                                 ctypes.byref(ln)))
    return out[:ln.value].copy()


def hf_critical_paths(g: Graph, s: int, delays, at, t_req, k: int, max_len: int, endpoints,
                      path, path_len):
    """NEXT-1 top-K endpoints per scenario (device tensors, stream-ordered): endpoints
    [S][K] int32 (or None), path [S][K][max_len] int32, path_len [S][K] int32."""
    tr = t_req if _is_torch(t_req) else None
    ts = 0.0 if _is_torch(t_req) else float(t_req)
    _check(_lib.hf_critical_paths_d(g.handle, s, _ptr(delays), _ptr(at), _ptr(tr),
                                    ctypes.c_float(ts), k, max_len, _ptr(endpoints), _ptr(path),
                                    _ptr(path_len)))
    return endpoints, path, path_len


def hf_mis(g: Graph, prio, in_set=None):
    """NEXT-4 greedy MIS (reading R19).  Host: prio numpy int32 [n] -> uint8 [n].
    Device: prio int32 CUDA tensor, in_set uint8 CUDA tensor (stream-ordered)."""
    if _is_torch(prio):
        _check(_lib.hf_mis_d(g.handle, _ptr(prio), _ptr(in_set)))
        return in_set
    p = _np(prio, np.int32)
    n = p.shape[0]
    out = np.zeros(max(n, 1), np.uint8)
    _check(_lib.hf_mis(g.handle, _ptr(p), _ptr(out)))
    return out[:n]


def hf_run_batch(g: Graph, s_local: int, delays, layout: int, t_req, at_src, wns_local,
                 nccl_comm=None, wns_all=None, at=None, rat=None):
    if _is_torch(delays):
        _check(_lib.hf_run_batch_d(g.handle, s_local, _ptr(delays), layout, _ptr(t_req),
                                   _ptr(at_src), _ptr(wns_local), _ptr(at), _ptr(rat),
                                   nccl_comm, _ptr(wns_all)))
    else:
        if at is not None or rat is not None:
            raise ValueError("at/rat outputs are only available with device tensors")
        _out(wns_local, s_local, np.float32, "wns_local")
        _out(wns_all, s_local, np.float32, "wns_all")
        d = _np(delays, np.float32)
        t = _np(t_req, np.float32)
        a = _np(at_src, np.float32)
        _check(_lib.hf_run_batch(g.handle, s_local, _ptr(d), layout, _ptr(t), _ptr(a),
                                 _ptr(wns_local), nccl_comm, _ptr(wns_all)))


def hf_analyze(n, m, fanin_ptr, fanin_src, s_local: int, delays, t_req, at_src, wns_local,
               delay=None, device: int = 0, stream=None, keep_graph: bool = False):
    """Create + levelize + batch in one call from host arrays (scenario data uploaded
    while the graph is built).  Returns (num_levels, Graph or None)."""
    _out(wns_local, s_local, np.float32, "wns_local")
    a = [_np(fanin_ptr, np.int32), _np(fanin_src, np.int32), _np(delay, np.float32)]
    d = _np(delays, np.float32)
    t = _np(t_req, np.float32)
    at = _np(at_src, np.float32)
    L = ctypes.c_int32()
    out = ctypes.c_void_p()
    _check(_lib.hf_analyze(n, m, _ptr(a[0]), _ptr(a[1]), _ptr(a[2]), s_local, _ptr(d), _ptr(t),
                           _ptr(at), _ptr(wns_local), ctypes.byref(L), device, _stream_of(stream),
                           ctypes.byref(out) if keep_graph else None))
    return L.value, (Graph(out, n, m, device) if keep_graph else None)


def hf_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.hf_nccl_unique_id(buf))
    return buf.raw


def hf_nccl_comm_init(uid: bytes, rank: int, nranks: int, device: int) -> ctypes.c_void_p:
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    comm = ctypes.c_void_p()
    _check(_lib.hf_nccl_comm_init(buf, rank, nranks, device, ctypes.byref(comm)))
    return comm


def hf_nccl_comm_destroy(comm):
    _check(_lib.hf_nccl_comm_destroy(comm))


def hf_profile_enable(g: Graph, on: bool = True):
    _check(_lib.hf_profile_enable(g.handle, 1 if on else 0))


def hf_profile_read(g: Graph):
    """(ms_levelize, ms_forward, ms_backward, kernel_launches)"""
    a, b, c = ctypes.c_float(), ctypes.c_float(), ctypes.c_float()
    k = ctypes.c_int64()
    _check(_lib.hf_profile_read(g.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                ctypes.byref(k)))
    return a.value, b.value, c.value, k.value


def hf_profile_read_batch(g: Graph) -> float:
    """ms of the propagation phase of the most recent hf_run_batch (fwd || bwd + slack)"""
    a = ctypes.c_float()
    _check(_lib.hf_profile_read_batch(g.handle, ctypes.byref(a)))
    return a.value


def hf_version() -> int:
    return _lib.hf_version()
