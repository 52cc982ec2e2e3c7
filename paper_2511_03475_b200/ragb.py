"""Thin Python binding of libragb's C-ABI (include/ragb.h).

Argument marshalling only: every step of the index build runs inside the
library (CUDA kernels for a1-a5, C++ for a6-a8).  PyTorch supplies device
memory and streams.  There is no fallback: if libragb.so is missing or has no
GPU to run on, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from fractions import Fraction

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", f"libragb_{os.environ['RAGB_LIB']}.so" if os.environ.get("RAGB_LIB")
                        else "libragb.so")

RB_OK, RB_EINVAL, RB_EDUPDOC, RB_EALPHA, RB_ENOMEM, RB_ECUDA, RB_ENCCL, RB_EPATH, RB_ESESSION, \
    RB_ESTATE = 0, -1, -2, -3, -4, -5, -6, -7, -8, -9
RB_EMIT_COUNTS, RB_ALPHA_ANY, RB_KEEP_ROWS, RB_SKIP_LINKAGE, RB_ASYNC_HOST = 1, 2, 4, 8, 16
RB_LINK_COMPLETE, RB_LINK_INTERSECTION = 0, 1
RB_CACHE_APPENDED, RB_CACHE_ACCESSED, RB_CACHE_EVICTED = 0, 1, 2
RB_PATH_GATHER, RB_PATH_GATHER_WIDE, RB_PATH_WINDOW, RB_PATH_WINDOW_WIDE, RB_PATH_INPLACE, \
    RB_PATH_CLIQUE_WARP, RB_PATH_CLIQUE_BLOCK = 1, 2, 4, 8, 16, 32, 64

STATUS_NAMES = {0: "RB_OK", -1: "RB_EINVAL", -2: "RB_EDUPDOC", -3: "RB_EALPHA", -4: "RB_ENOMEM",
                -5: "RB_ECUDA", -6: "RB_ENCCL", -7: "RB_EPATH", -8: "RB_ESESSION", -9: "RB_ESTATE"}

EXPORTED = [
    "rb_version", "rb_last_error", "rb_params_init", "rb_workspace_size", "rb_build_index",
    "rb_build_index_host", "rb_index_from_linkage", "rb_index_size", "rb_index_stats", "rb_index_shard",
    "rb_index_wait",
    "rb_index_counts", "rb_index_nn",
    "rb_index_linkage", "rb_index_tree_info", "rb_index_tree", "rb_order_contexts", "rb_session_open",
    "rb_session_open_docs", "rb_dedup_turn", "rb_session_turn", "rb_session_free", "rb_index_free",
    "rb_index_set_alpha", "rb_index_set_online", "rb_session_context", "rb_dedup_batch",
    "rb_index_cache_event", "rb_index_cache_state", "rb_cache_create", "rb_cache_prefill",
    "rb_cache_prefill_batch", "rb_cache_resident", "rb_cache_free",
    "rb_dist_create", "rb_dist_workspace_size", "rb_dist_attach", "rb_dist_export", "rb_dist_import",
    "rb_build_index_dist", "rb_dist_free",
]


class RagbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


class Params(ctypes.Structure):
    _fields_ = [("alpha_num", ctypes.c_uint32), ("alpha_den", ctypes.c_uint32),
                ("linkage", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("stream", ctypes.c_void_p), ("row0", ctypes.c_int64), ("nrows", ctypes.c_int64),
                # implementation strategy (ragb.h): no result depends on it
                ("value_codes", ctypes.c_int32), ("inplace", ctypes.c_int32),
                ("inplace_weight", ctypes.c_float), ("gather", ctypes.c_int32),
                ("long_lists", ctypes.c_int32), ("dist_grid", ctypes.c_int32),
                ("host_threads", ctypes.c_int32), ("trace", ctypes.c_int32),
                ("side_buffer", ctypes.c_int32), ("nn_cache", ctypes.c_int32)]

TUNING_FIELDS = ("value_codes", "inplace", "inplace_weight", "gather", "long_lists", "dist_grid",
                 "host_threads", "trace", "side_buffer", "nn_cache")


class Stats(ctypes.Structure):
    _fields_ = [("validate_ms", ctypes.c_float), ("distance_ms", ctypes.c_float),
                ("linkage_ms", ctypes.c_float), ("host_ms", ctypes.c_float),
                ("total_ms", ctypes.c_float), ("linkage_rounds", ctypes.c_int32),
                ("kernel_launches", ctypes.c_int32), ("n_virtual", ctypes.c_int64),
                ("max_depth", ctypes.c_int64), ("merge_ms", ctypes.c_float),
                ("merge_launches", ctypes.c_int32), ("merge_bytes", ctypes.c_double),
                ("value_codes", ctypes.c_int32), ("max_level", ctypes.c_int32),
                ("paths", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load libragb.so (built by paper_2511_03475_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libragb.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    P, i64, i32, u32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_size_t
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "rb_version": ([], ctypes.c_char_p),
        "rb_last_error": ([], ctypes.c_char_p),
        "rb_params_init": ([ctypes.POINTER(Params)], i32),
        "rb_workspace_size": ([i64, i32, ctypes.POINTER(Params), ctypes.POINTER(sz), ctypes.POINTER(sz)], i32),
        "rb_build_index": ([P, P, i64, i32, ctypes.POINTER(Params), P, P, sz, P, P, PP], i32),
        "rb_build_index_host": ([P, P, i64, i32, ctypes.POINTER(Params), P, P, sz, PP], i32),
        "rb_index_from_linkage": ([P, P, i64, i32, P, P, P, P, PP], i32),
        "rb_index_size": ([P, ctypes.POINTER(i64), ctypes.POINTER(i32)], i32),
        "rb_index_stats": ([P, ctypes.POINTER(Stats)], i32),
        "rb_index_wait": ([P], i32),
        "rb_index_shard": ([P, ctypes.POINTER(i64), ctypes.POINTER(i64)], i32),
        "rb_index_counts": ([P, i64, i64, P, P], i32),
        "rb_index_nn": ([P, P, P], i32),
        "rb_index_linkage": ([P, P, P, P, P], i32),
        "rb_index_tree_info": ([P, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)], i32),
        "rb_index_tree": ([P, P, P, P, P, P, P, P], i32),
        "rb_order_contexts": ([P, P, P, i64, i32, P, P, P], i32),
        "rb_index_set_alpha": ([P, u32, u32], i32),
        "rb_index_set_online": ([P, i32], i32),
        "rb_session_context": ([P, P, i32, ctypes.POINTER(i32)], i32),
        "rb_dedup_batch": ([P, i64, P, P, P, i64, i32, P, P, P, P, P], i32),
        "rb_index_cache_event": ([P, i32, P, i32, i64, ctypes.POINTER(i64)], i32),
        "rb_index_cache_state": ([P, P, P], i32),
        "rb_cache_create": ([i64, PP], i32),
        "rb_cache_prefill": ([P, P, i32, P, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)], i32),
        "rb_cache_prefill_batch": ([P, P, P, P, i64, i32, i32, P, P, P], i32),
        "rb_cache_resident": ([P, ctypes.POINTER(i64)], i32),
        "rb_cache_free": ([P], None),
        "rb_dist_create": ([i32, i32, i32, PP], i32),
        "rb_dist_workspace_size": ([i32, i64, i32, ctypes.POINTER(sz), ctypes.POINTER(sz)], i32),
        "rb_dist_attach": ([P, i32, P, P, sz], i32),
        "rb_dist_export": ([P, P, sz], i32),
        "rb_dist_import": ([P, P, sz], i32),
        "rb_build_index_dist": ([P, P, P, i64, i32, ctypes.POINTER(Params), PP], i32),
        "rb_dist_free": ([P], None),
        "rb_session_open": ([P, i64, PP], i32),
        "rb_session_open_docs": ([P, i32, PP], i32),
        "rb_dedup_turn": ([P, P, i32, P, ctypes.POINTER(i32), P, P, ctypes.POINTER(i32)], i32),
        "rb_session_turn": ([P, ctypes.POINTER(i32)], i32),
        "rb_session_free": ([P], None),
        "rb_index_free": ([P], None),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(rc: int):
    if rc != RB_OK:
        raise RagbError(rc, lib().rb_last_error().decode())


def _np_ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def version() -> str:
    return lib().rb_version().decode()


def alpha_rational(alpha) -> tuple[int, int]:
    """X1: alpha as an exact rational with denominator <= 1000."""
    if isinstance(alpha, tuple):
        return int(alpha[0]), int(alpha[1])
    f = Fraction(alpha).limit_denominator(1000)
    return f.numerator, f.denominator


def make_params(alpha=(1, 200), flags=0, stream=None, row0=0, nrows=-1, linkage=RB_LINK_COMPLETE,
                tuning: dict | None = None) -> Params:
    """tuning: implementation-strategy fields of rb_params (TUNING_FIELDS);
    the library's automatic choice where absent."""
    p = Params()
    _check(lib().rb_params_init(ctypes.byref(p)))
    p.alpha_num, p.alpha_den = alpha_rational(alpha)
    p.linkage = linkage
    p.flags = flags
    p.stream = stream
    p.row0 = row0
    p.nrows = nrows
    for k, v in (tuning or {}).items():
        if k not in TUNING_FIELDS:
            raise KeyError(f"unknown tuning field {k!r}")
        setattr(p, k, v)
    return p


def workspace_size(N: int, K: int, params: Params) -> tuple[int, int]:
    rb, sb = ctypes.c_size_t(), ctypes.c_size_t()
    _check(lib().rb_workspace_size(N, K, ctypes.byref(params), ctypes.byref(rb), ctypes.byref(sb)))
    return rb.value, sb.value


class Index:
    """Owns an rb_index handle (host results of one build)."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        n, k = ctypes.c_int64(), ctypes.c_int32()
        _check(lib().rb_index_size(self._h, ctypes.byref(n), ctypes.byref(k)))
        self.N, self.K = n.value, k.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.rb_index_free(h)
            self._h = None

    def wait(self):
        """RB_ASYNC_HOST builds: wait for the host stage (a6-a7); every other
        method waits by itself."""
        _check(lib().rb_index_wait(self._h))
        return self

    def stats(self) -> dict:
        s = Stats()
        _check(lib().rb_index_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def shard(self):
        """(row0, nrows): the distance rows this index was built for."""
        r0, nr = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().rb_index_shard(self._h, ctypes.byref(r0), ctypes.byref(nr)))
        return r0.value, nr.value

    def counts(self, row0=0, nrows=None, device="cuda"):
        """Parity output: (s uint8, D int16 viewed as uint16) [nrows][N] device
        tensors of Eq. 1's overlap and positional sum for rows row0.."""
        import torch
        n = self.N - row0 if nrows is None else nrows
        s = torch.empty((n, self.N), dtype=torch.uint8, device=device)
        D = torch.empty((n, self.N), dtype=torch.int16, device=device)
        _check(lib().rb_index_counts(self._h, row0, n, ctypes.c_void_p(s.data_ptr()), ctypes.c_void_p(D.data_ptr())))
        return s, D

    def nn(self, nrows=None):
        n = self.N if nrows is None else nrows
        idx = np.empty(n, dtype=np.int32)
        val = np.empty(n, dtype=np.float32)
        _check(lib().rb_index_nn(self._h, _np_ptr(idx), _np_ptr(val)))
        return idx, val

    def linkage(self):
        n = max(self.N - 1, 0)
        a, b, s = (np.empty(n, dtype=np.int32) for _ in range(3))
        h = np.empty(n, dtype=np.float32)
        _check(lib().rb_index_linkage(self._h, _np_ptr(a), _np_ptr(b), _np_ptr(h), _np_ptr(s)))
        return a, b, h, s

    def tree(self) -> dict:
        nn_, pt, qt = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().rb_index_tree_info(self._h, ctypes.byref(nn_), ctypes.byref(pt), ctypes.byref(qt)))
        n = nn_.value
        parent, leaf, rep = (np.empty(n, dtype=np.int32) for _ in range(3))
        poff = np.empty(n + 1, dtype=np.int64)
        pids = np.empty(pt.value, dtype=np.uint32)
        qoff = np.empty(self.size() + 1, dtype=np.int64)
        path = np.empty(qt.value, dtype=np.int32)
        _check(lib().rb_index_tree(self._h, _np_ptr(parent), _np_ptr(leaf), _np_ptr(rep), _np_ptr(poff),
                                   _np_ptr(pids), _np_ptr(qoff), _np_ptr(path)))
        return dict(parent=parent, leaf=leaf, rep=rep, prefix_off=poff, prefix_ids=pids,
                    path_off=qoff, path=path)

    def size(self) -> int:
        n, k = ctypes.c_int64(), ctypes.c_int32()
        _check(lib().rb_index_size(self._h, ctypes.byref(n), ctypes.byref(k)))
        return n.value

    def paths(self):
        t = self.tree()
        o, p = t["path_off"], t["path"]
        return [p[o[i]:o[i + 1]].tolist() for i in range(len(o) - 1)]

    def cache_event(self, kind, path=(), n_tokens=0) -> int:
        """NEXT-4: Appended / Accessed / Evicted; returns the
        tokens evicted (Evicted) or 0."""
        pa = np.ascontiguousarray(list(path), dtype=np.int32)
        taken = ctypes.c_int64()
        _check(lib().rb_index_cache_event(self._h, kind, _np_ptr(pa) if len(pa) else None, len(pa), n_tokens,
                                          ctypes.byref(taken)))
        return taken.value

    def cache_state(self):
        n = len(self.tree()["parent"])
        seq = np.empty(n, dtype=np.int64)
        last = np.empty(n, dtype=np.int64)
        _check(lib().rb_index_cache_state(self._h, _np_ptr(seq), _np_ptr(last)))
        return seq, last

    def set_online(self, device: int):
        """NEXT-1 root scoring: 1 GPU, 0 host, -1 auto (rb_index_set_online)."""
        _check(lib().rb_index_set_online(self._h, int(device)))

    def set_alpha(self, alpha):
        an, ad = alpha_rational(alpha)
        _check(lib().rb_index_set_alpha(self._h, an, ad))

    def order_new(self, ids, lens=None):
        """NEXT-1: search + insert + order new contexts (host [M, K]); returns
        (ordered [M, K], prefix_len [M], schedule [M])."""
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        M, K = ids.shape
        lens_a = None if lens is None else np.ascontiguousarray(lens, dtype=np.uint8)
        out = np.empty((M, K), dtype=np.uint32)
        plen = np.empty(M, dtype=np.uint8)
        sched = np.empty(M, dtype=np.int64)
        _check(lib().rb_order_contexts(self._h, _np_ptr(ids), _np_ptr(lens_a), M, K, _np_ptr(out),
                                       _np_ptr(plen), _np_ptr(sched)))
        return out, plen, sched

    def order_contexts(self, out=None):
        """Offline prefix-first ordering + schedule of the indexed set.
        ``out``: optional (ordered [n][K] uint32, prefix_len [n] uint8,
        schedule [n] int64) arrays to fill (reused across calls)."""
        n = self.size()
        if out is None:
            out, plen, sched = (np.empty((n, self.K), dtype=np.uint32), np.empty(n, dtype=np.uint8),
                                np.empty(n, dtype=np.int64))
        else:
            out, plen, sched = out
            if (out.shape != (n, self.K) or out.dtype != np.uint32 or plen.shape != (n,) or plen.dtype != np.uint8
                    or sched.shape != (n,) or sched.dtype != np.int64
                    or not all(a.flags.c_contiguous for a in (out, plen, sched))):
                raise ValueError("order_contexts: out arrays must be C-contiguous uint32 [n][K], uint8 [n], int64 [n]")
        _check(lib().rb_order_contexts(self._h, None, None, n, self.K, _np_ptr(out), _np_ptr(plen),
                                       _np_ptr(sched)))
        return out, plen, sched

    def session(self, row: int) -> "Session":
        h = ctypes.c_void_p()
        _check(lib().rb_session_open(self._h, row, ctypes.byref(h)))
        return Session(h, keepalive=self)


class Session:
    """Multi-turn de-duplication state."""

    def __init__(self, handle, keepalive=None):
        self._h = handle
        self._keep = keepalive

    @classmethod
    def from_docs(cls, docs) -> "Session":
        d = np.ascontiguousarray(docs, dtype=np.uint32)
        h = ctypes.c_void_p()
        _check(lib().rb_session_open_docs(_np_ptr(d), d.shape[0], ctypes.byref(h)))
        return cls(h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.rb_session_free(h)
            self._h = None

    @property
    def turn(self) -> int:
        t = ctypes.c_int32()
        _check(lib().rb_session_turn(self._h, ctypes.byref(t)))
        return t.value

    def dedup_turn(self, docs):
        d = np.ascontiguousarray(docs, dtype=np.uint32)
        n = d.shape[0]
        novel = np.empty(max(n, 1), dtype=np.uint32)
        rdoc = np.empty(max(n, 1), dtype=np.uint32)
        rturn = np.empty(max(n, 1), dtype=np.int32)
        nn_, nr = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().rb_dedup_turn(self._h, _np_ptr(d), n, _np_ptr(novel), ctypes.byref(nn_), _np_ptr(rdoc),
                                   _np_ptr(rturn), ctypes.byref(nr)))
        return novel[:nn_.value].copy(), rdoc[:nr.value].copy(), rturn[:nr.value].copy()

    def context(self) -> np.ndarray:
        """Cumulative context: turn-0 docs ++ every turn's novel docs."""
        n = ctypes.c_int32()
        _check(lib().rb_session_context(self._h, None, 0, ctypes.byref(n)))
        out = np.empty(max(n.value, 1), dtype=np.uint32)
        _check(lib().rb_session_context(self._h, _np_ptr(out), n.value, ctypes.byref(n)))
        return out[:n.value].copy()


def dedup_batch(sessions, turn_session, ids, lens=None):
    """NEXT-2: row i is the next turn of sessions[turn_session[i]]; returns
    (novel [M,K], n_novel [M], ref_doc [M,K], ref_turn [M,K], n_ref [M])."""
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    M, K = ids.shape
    ts = np.ascontiguousarray(turn_session, dtype=np.int64)
    lens_a = None if lens is None else np.ascontiguousarray(lens, dtype=np.uint8)
    handles = (ctypes.c_void_p * max(len(sessions), 1))(*[s._h.value if hasattr(s._h, "value") else s._h
                                                          for s in sessions])
    novel = np.empty((M, K), dtype=np.uint32)
    rdoc = np.empty((M, K), dtype=np.uint32)
    rturn = np.empty((M, K), dtype=np.int32)
    nn_ = np.empty(M, dtype=np.int32)
    nr = np.empty(M, dtype=np.int32)
    _check(lib().rb_dedup_batch(handles, len(sessions), _np_ptr(ts), _np_ptr(ids), _np_ptr(lens_a), M, K,
                                _np_ptr(novel), _np_ptr(nn_), _np_ptr(rdoc), _np_ptr(rturn), _np_ptr(nr)))
    return novel, nn_, rdoc, rturn, nr


def index_from_linkage(ids, a, b, h, size, lens=None) -> Index:
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    N, K = ids.shape
    arrs = [np.ascontiguousarray(x, dtype=t) for x, t in
            ((a, np.int32), (b, np.int32), (h, np.float32), (size, np.int32))]
    lens_a = None if lens is None else np.ascontiguousarray(lens, dtype=np.uint8)
    out = ctypes.c_void_p()
    _check(lib().rb_index_from_linkage(_np_ptr(ids), _np_ptr(lens_a), N, K, *[_np_ptr(x) for x in arrs],
                                       ctypes.byref(out)))
    return Index(out)


# ---------------------------------------------------------------- device path
class Workspace:
    """Caller-owned device buffers (torch allocations) for one (N, K, flags)."""

    def __init__(self, N, K, params: Params, device="cuda"):
        import torch
        self.N, self.K = N, K
        rb, sb = workspace_size(N, K, params)
        nrows = rb // (4 * N)
        self.rows = torch.empty((nrows, N), dtype=torch.float32, device=device)
        self.scratch = torch.empty(max(sb, 1), dtype=torch.uint8, device=device)
        self.s = self.D = None
        if params.flags & RB_EMIT_COUNTS:
            self.s = torch.empty((nrows, N), dtype=torch.uint8, device=device)
            self.D = torch.empty((nrows, N), dtype=torch.int16, device=device)


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def build_index(ids, lens=None, *, alpha=(1, 200), flags=0, row0=0, nrows=-1, stream=None,
                workspace: Workspace | None = None, linkage=RB_LINK_COMPLETE, tuning: dict | None = None):
    """Build the context index from device ids (torch.int32/uint32 CUDA tensor [N, K]).

    Returns (Index, Workspace); workspace.rows holds the distance rows (unless
    the linkage consumed them: pass flags |= RB_KEEP_ROWS to keep them).
    flags |= RB_ASYNC_HOST returns once the device stages are done (the
    workspace is free for the next build) and finishes the tree / orders /
    schedule on a library thread; Index methods wait for it (ragb.h
    rb_index_wait)."""
    import torch
    if not ids.is_cuda:
        raise ValueError("build_index expects a CUDA tensor; use build_index_host for host arrays")
    if ids.dtype not in (torch.int32, torch.uint32):
        raise TypeError("ids must be int32/uint32 (bit pattern of uint32 DocIds)")
    ids = ids.contiguous()
    N, K = ids.shape
    p = make_params(alpha, flags, _stream_ptr(stream), row0, nrows, linkage, tuning)
    ws = workspace or Workspace(N, K, p, device=ids.device)
    if lens is not None:
        lens = lens.contiguous()
        assert lens.dtype == torch.uint8 and lens.is_cuda
    out = ctypes.c_void_p()
    _check(lib().rb_build_index(
        ctypes.c_void_p(ids.data_ptr()), None if lens is None else ctypes.c_void_p(lens.data_ptr()), N, K,
        ctypes.byref(p), ctypes.c_void_p(ws.rows.data_ptr()), ctypes.c_void_p(ws.scratch.data_ptr()),
        ws.scratch.numel(), None if ws.s is None else ctypes.c_void_p(ws.s.data_ptr()),
        None if ws.D is None else ctypes.c_void_p(ws.D.data_ptr()), ctypes.byref(out)))
    return Index(out), ws


def build_index_host(ids, lens=None, *, alpha=(1, 200), flags=0, stream=None,
                     workspace: Workspace | None = None, linkage=RB_LINK_COMPLETE, tuning: dict | None = None):
    """End-to-end entry: ids/lens are host numpy arrays; H2D happens inside."""
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    N, K = ids.shape
    p = make_params(alpha, flags, _stream_ptr(stream), linkage=linkage, tuning=tuning)
    ws = workspace or Workspace(N, K, p)
    lens_a = None if lens is None else np.ascontiguousarray(lens, dtype=np.uint8)
    out = ctypes.c_void_p()
    _check(lib().rb_build_index_host(_np_ptr(ids), _np_ptr(lens_a), N, K, ctypes.byref(p),
                                     ctypes.c_void_p(ws.rows.data_ptr()), ctypes.c_void_p(ws.scratch.data_ptr()),
                                     ws.scratch.numel(), ctypes.byref(out)))
    return Index(out), ws


class PrefixCache:
    """NEXT-4: document-granularity prefix cache."""

    def __init__(self, capacity_tokens: int):
        h = ctypes.c_void_p()
        _check(lib().rb_cache_create(int(capacity_tokens), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.rb_cache_free(h)
            self._h = None

    def prefill(self, docs, doc_tokens=None):
        d = np.ascontiguousarray(docs, dtype=np.uint32)
        t = None if doc_tokens is None else np.ascontiguousarray(doc_tokens, dtype=np.int32)
        hit, miss, ev = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().rb_cache_prefill(self._h, _np_ptr(d), d.shape[0], _np_ptr(t), ctypes.byref(hit),
                                      ctypes.byref(miss), ctypes.byref(ev)))
        return hit.value, miss.value, ev.value

    def prefill_batch(self, ids, lens=None, order=None, tokens_per_doc=1):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        M, K = ids.shape
        lens_a = None if lens is None else np.ascontiguousarray(lens, dtype=np.uint8)
        ord_a = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
        hit = np.empty(M, dtype=np.int64)
        miss = np.empty(M, dtype=np.int64)
        ev = np.empty(M, dtype=np.int64)
        _check(lib().rb_cache_prefill_batch(self._h, _np_ptr(ids), _np_ptr(lens_a), _np_ptr(ord_a), M, K,
                                            tokens_per_doc, _np_ptr(hit), _np_ptr(miss), _np_ptr(ev)))
        return hit, miss, ev

    @property
    def resident(self) -> int:
        r = ctypes.c_int64()
        _check(lib().rb_cache_resident(self._h, ctypes.byref(r)))
        return r.value


RB_DIST_HANDLE_BYTES = 256


class DistBuilder:
    """§8(e): one index built by `world` GPUs with the distance rows sharded.

    local=True: all ranks in this process on the current device (validation
    of the sharded algorithm on one GPU).  local=False: one process per GPU
    (torchrun); the handle blobs are exchanged with torch.distributed.
    """

    def __init__(self, world: int, N: int, K: int, rank: int = 0, local: bool = False, device="cuda"):
        import torch
        self.world, self.N, self.K, self.rank, self.local = world, N, K, rank, local
        h = ctypes.c_void_p()
        _check(lib().rb_dist_create(world, rank, world if local else 1, ctypes.byref(h)))
        self._h = h
        rb, sb = ctypes.c_size_t(), ctypes.c_size_t()
        _check(lib().rb_dist_workspace_size(world, N, K, ctypes.byref(rb), ctypes.byref(sb)))
        ranks = range(world) if local else [rank]
        self.rows, self.scratch = {}, {}
        for q in ranks:
            self.rows[q] = torch.empty(max(rb.value // 4, 1), dtype=torch.float32, device=device)
            self.scratch[q] = torch.empty(sb.value, dtype=torch.uint8, device=device)
            _check(lib().rb_dist_attach(self._h, q, ctypes.c_void_p(self.rows[q].data_ptr()),
                                        ctypes.c_void_p(self.scratch[q].data_ptr()), sb.value))
        if not local and world > 1:
            import torch.distributed as dist
            blob = ctypes.create_string_buffer(RB_DIST_HANDLE_BYTES)
            _check(lib().rb_dist_export(self._h, blob, RB_DIST_HANDLE_BYTES))
            blobs = [None] * world
            dist.all_gather_object(blobs, bytes(blob.raw))
            for b in blobs:
                buf = ctypes.create_string_buffer(b, RB_DIST_HANDLE_BYTES)
                _check(lib().rb_dist_import(self._h, buf, RB_DIST_HANDLE_BYTES))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.rb_dist_free(h)
            self._h = None

    def build(self, ids, lens=None, *, alpha=(1, 200), flags=0, stream=None, tuning: dict | None = None) -> Index:
        ids = ids.contiguous()
        N, K = ids.shape
        assert (N, K) == (self.N, self.K)
        p = make_params(alpha, flags, _stream_ptr(stream), tuning=tuning)
        out = ctypes.c_void_p()
        _check(lib().rb_build_index_dist(self._h, ctypes.c_void_p(ids.data_ptr()),
                                         None if lens is None else ctypes.c_void_p(lens.contiguous().data_ptr()),
                                         N, K, ctypes.byref(p), ctypes.byref(out)))
        return Index(out)


def torch_cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
