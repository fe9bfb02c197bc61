"""Thin ctypes binding of liba2ats.so (include/a2ats.h).

Argument marshalling only: every step of the retrieval path runs in the CUDA
kernels behind the C ABI.  Torch tensors are accepted for convenience (device,
dtype and contiguity are checked, then ``data_ptr()`` is passed); there is no
CPU fallback -- if the library cannot be loaded every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

PKG = os.path.dirname(os.path.abspath(__file__))
# A2ATS_LIB selects a tuning variant built by build.build_variant (tools only)
LIB_PATH = os.environ.get("A2ATS_LIB") or os.path.join(PKG, "lib", "liba2ats.so")

A2ATS_OK = 0
A2ATS_EINVAL = -1
A2ATS_EUNSUPPORTED = -2
A2ATS_EWORKSPACE = -3
A2ATS_ECUDA = -4
A2ATS_ENCCL = -5
A2ATS_GROUP_MAX = 0
A2ATS_GROUP_SUM = 1
A2ATS_GROUP_PER_HEAD = 2
A2ATS_ROPE_WINDOWED = 0
A2ATS_ROPE_STANDARD = 1
A2ATS_KV_DEVICE = 0
A2ATS_KV_HOST_MAPPED = 1
A2ATS_LUT_AUTO, A2ATS_LUT_TENSOR, A2ATS_LUT_FMA = 0, 1, 2


class A2ATSError(RuntimeError):
    def __init__(self, fn: str, status: int):
        self.status = status
        extra = ""
        if status == A2ATS_ECUDA:
            extra = " [" + load().a2ats_last_cuda_error().decode() + "]"
        super().__init__(f"{fn} -> {status}: {status_string(status)}{extra}")


class a2ats_shape(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("Hq", ctypes.c_int32), ("Hkv", ctypes.c_int32),
                ("d", ctypes.c_int32), ("L", ctypes.c_int32), ("n_max", ctypes.c_int32),
                ("code_bytes", ctypes.c_int32)]


class a2ats_params(ctypes.Structure):
    _fields_ = [("window", ctypes.c_int32), ("bridge", ctypes.c_int32), ("n_sink", ctypes.c_int32),
                ("topk", ctypes.c_int32), ("rope_theta", ctypes.c_double),
                ("inv_freq", ctypes.POINTER(ctypes.c_double)), ("group_reduce", ctypes.c_int32),
                ("kv_location", ctypes.c_int32), ("lut_engine", ctypes.c_int32), ("hist_lag", ctypes.c_int32),
                ("rope_mode", ctypes.c_int32)]


_VP = ctypes.c_void_p
_SIGS = {
    "a2ats_default_params": (None, [ctypes.POINTER(a2ats_params)]),
    "a2ats_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "a2ats_abi_version": (ctypes.c_int, []),
    "a2ats_stage_rows": (ctypes.c_int, [ctypes.POINTER(a2ats_shape), ctypes.c_int32, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "a2ats_last_cuda_error": (ctypes.c_char_p, []),
    "a2ats_qavq_prepare": (ctypes.c_int, [ctypes.POINTER(a2ats_shape), _VP, _VP, _VP, _VP, _VP]),
    "a2ats_build_codes_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(a2ats_shape)]),
    "a2ats_build_codes": (ctypes.c_int, [ctypes.POINTER(a2ats_shape), _VP, ctypes.c_int32, ctypes.c_int32, _VP, _VP,
                                         _VP, _VP, _VP, ctypes.c_size_t, _VP]),
    "a2ats_decode_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(a2ats_shape), ctypes.POINTER(a2ats_params)]),
    "a2ats_set_stage_events": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int]),
    "a2ats_decode_step": (ctypes.c_int, [ctypes.POINTER(a2ats_shape), ctypes.POINTER(a2ats_params), ctypes.c_int32,
                                         _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, ctypes.c_size_t, _VP]),
    "a2ats_decode_step_append": (ctypes.c_int, [ctypes.POINTER(a2ats_shape), ctypes.POINTER(a2ats_params),
                                                ctypes.c_int32, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                                _VP, _VP, ctypes.c_size_t, _VP]),
    "a2ats_select_topk": (ctypes.c_int, [ctypes.POINTER(a2ats_shape), ctypes.POINTER(a2ats_params), ctypes.c_int32,
                                         _VP, _VP, _VP, _VP, _VP, _VP, ctypes.c_size_t, _VP]),
}

_lib = None


ABI_VERSION = 10  # include/a2ats.h A2ATS_ABI_VERSION


def load(path: str = LIB_PATH, build_if_missing: bool = True) -> ctypes.CDLL:
    """Load (building first if needed) liba2ats.so and declare its signatures."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path) and build_if_missing:
        from .build import build
        build()
    if not os.path.exists(path):
        raise OSError(f"liba2ats.so not found at {path}: run `python -m paper_2502_12665_b200.build`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    if lib.a2ats_abi_version() != ABI_VERSION:
        raise OSError(f"{path}: ABI version {lib.a2ats_abi_version()}, binding expects {ABI_VERSION}; rebuild it")
    _lib = lib
    return lib


def status_string(status: int) -> str:
    return load().a2ats_status_string(status).decode()


def _check(fn: str, rc: int):
    if rc != A2ATS_OK:
        raise A2ATSError(fn, rc)


# ------------------------------------------------------------------ shapes / params
def make_shape(B, Hq, Hkv, d, L, n_max, code_bytes=2) -> a2ats_shape:
    return a2ats_shape(B, Hq, Hkv, d, L, n_max, code_bytes)


@dataclass
class Params:
    window: int = 64
    bridge: int = 2048
    n_sink: int = 4
    topk: int = 0
    rope_theta: float = 1e4
    inv_freq: tuple | None = None
    group_reduce: int = A2ATS_GROUP_MAX
    kv_location: int = A2ATS_KV_DEVICE
    lut_engine: int = A2ATS_LUT_AUTO
    hist_lag: int = 0
    rope_mode: int = 0  # A2ATS_ROPE_WINDOWED | A2ATS_ROPE_STANDARD

    def c(self) -> a2ats_params:
        p = a2ats_params()
        load().a2ats_default_params(ctypes.byref(p))
        p.window, p.bridge, p.n_sink, p.topk = self.window, self.bridge, self.n_sink, self.topk
        p.rope_theta = self.rope_theta
        if self.inv_freq is not None:
            if len(self.inv_freq) != 64:  # the library reads d/2 = 64 doubles
                raise ValueError(f"inv_freq must hold d/2 = 64 frequencies, got {len(self.inv_freq)}")
            self._freq_buf = (ctypes.c_double * len(self.inv_freq))(*self.inv_freq)
            p.inv_freq = ctypes.cast(self._freq_buf, ctypes.POINTER(ctypes.c_double))
        p.group_reduce, p.kv_location, p.lut_engine = self.group_reduce, self.kv_location, self.lut_engine
        p.hist_lag = self.hist_lag
        p.rope_mode = self.rope_mode
        return p


def _ptr(t, name, dtype=None, optional=False, host_ok=False):
    if t is None:
        if optional:
            return None
        raise ValueError(f"{name} is required")
    if isinstance(t, int):
        return t
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if not t.is_cuda:
        if not host_ok:
            raise ValueError(f"{name} must be a CUDA tensor")
        if host_ok == "pinned" and not t.is_pinned():
            raise ValueError(f"{name}: host tensors must be pinned (mapped) memory")
    return t.data_ptr()


def _code_dtype(shape):
    import torch
    return torch.uint8 if getattr(shape, "code_bytes", 2) == 1 else torch.uint16


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


# ------------------------------------------------------------------ entry points (same names as the C ABI)
def a2ats_qavq_prepare(shape: a2ats_shape, codebook, H, nrm, chat, stream=None):
    import torch
    rc = load().a2ats_qavq_prepare(ctypes.byref(shape), _ptr(codebook, "codebook", torch.bfloat16),
                                   _ptr(H, "H", torch.float32, optional=True), _ptr(nrm, "nrm", torch.float32),
                                   _ptr(chat, "chat", torch.bfloat16), _stream(stream))
    _check("a2ats_qavq_prepare", rc)


def a2ats_build_codes_workspace_bytes(shape: a2ats_shape) -> int:
    return int(load().a2ats_build_codes_workspace_bytes(ctypes.byref(shape)))


def a2ats_build_codes(shape: a2ats_shape, keys, t_begin: int, t_end: int, chat, nrm, codes, hist, ws,
                      stream=None):
    import torch
    rc = load().a2ats_build_codes(ctypes.byref(shape), _ptr(keys, "keys", torch.bfloat16), int(t_begin), int(t_end),
                                  _ptr(chat, "chat", torch.bfloat16), _ptr(nrm, "nrm", torch.float32), _ptr(codes, "codes", _code_dtype(shape)),
                                  _ptr(hist, "hist", torch.int32, optional=True), _ptr(ws, "ws"),
                                  ws.numel() * ws.element_size(), _stream(stream))
    _check("a2ats_build_codes", rc)


def a2ats_decode_workspace_bytes(shape: a2ats_shape, params) -> int:
    p = params.c() if isinstance(params, Params) else params
    return int(load().a2ats_decode_workspace_bytes(ctypes.byref(shape), ctypes.byref(p)))


def a2ats_decode_step(shape: a2ats_shape, params, n_ctx: int, q, k_cache, v_cache, codes, codebook, hist, out,
                      sel_out, scores_out, ws, stream=None, kv_host: bool = False):
    import torch
    p = params.c() if isinstance(params, Params) else params
    rc = load().a2ats_decode_step(
        ctypes.byref(shape), ctypes.byref(p), int(n_ctx), _ptr(q, "q", torch.bfloat16),
        _ptr(k_cache, "k_cache", torch.bfloat16, host_ok=kv_host), _ptr(v_cache, "v_cache", torch.bfloat16, host_ok=kv_host),
        _ptr(codes, "codes", _code_dtype(shape)), _ptr(codebook, "codebook", torch.bfloat16),
        _ptr(hist, "hist", torch.int32, optional=True), _ptr(out, "out", torch.float32, host_ok="pinned"),
        _ptr(sel_out, "sel_out", torch.int32, optional=True), _ptr(scores_out, "scores_out", torch.float32, optional=True),
        _ptr(ws, "ws"), ws.numel() * ws.element_size(), _stream(stream))
    _check("a2ats_decode_step", rc)


def a2ats_decode_step_append(shape: a2ats_shape, params, n_ctx: int, q, k_cache, v_cache, codes, codebook, hist,
                             chat, nrm, out, sel_out, scores_out, ws, stream=None):
    import torch
    p = params.c() if isinstance(params, Params) else params
    rc = load().a2ats_decode_step_append(
        ctypes.byref(shape), ctypes.byref(p), int(n_ctx), _ptr(q, "q", torch.bfloat16),
        _ptr(k_cache, "k_cache", torch.bfloat16), _ptr(v_cache, "v_cache", torch.bfloat16),
        _ptr(codes, "codes", _code_dtype(shape)), _ptr(codebook, "codebook", torch.bfloat16),
        _ptr(hist, "hist", torch.int32, optional=True), _ptr(chat, "chat", torch.bfloat16),
        _ptr(nrm, "nrm", torch.float32), _ptr(out, "out", torch.float32, host_ok="pinned"),
        _ptr(sel_out, "sel_out", torch.int32, optional=True), _ptr(scores_out, "scores_out", torch.float32, optional=True),
        _ptr(ws, "ws"), ws.numel() * ws.element_size(), _stream(stream))
    _check("a2ats_decode_step_append", rc)


def a2ats_stage_rows(shape: a2ats_shape, n_ctx: int, q_src, k_src, v_src, q_dst, k_cache, v_cache, stream=None):
    """One kernel copies q and the new token's K/V rows (device or pinned host sources) into
    q_dst and row n_ctx - 1 of the caches."""
    import torch
    rc = load().a2ats_stage_rows(
        ctypes.byref(shape), int(n_ctx), _ptr(q_src, "q_src", torch.bfloat16, optional=True, host_ok="pinned"),
        _ptr(k_src, "k_src", torch.bfloat16, optional=True, host_ok="pinned"),
        _ptr(v_src, "v_src", torch.bfloat16, optional=True, host_ok="pinned"),
        _ptr(q_dst, "q_dst", torch.bfloat16, optional=True), _ptr(k_cache, "k_cache", torch.bfloat16, optional=True),
        _ptr(v_cache, "v_cache", torch.bfloat16, optional=True), _stream(stream))
    _check("a2ats_stage_rows", rc)


def a2ats_select_topk(shape: a2ats_shape, params, n_ctx: int, q, codes, codebook, hist, sel_out, ws, stream=None):
    """a1..a4 only (score table + top-K): Sel into sel_out [B, Hkv, K_eff] int32."""
    import torch
    p = params.c() if isinstance(params, Params) else params
    rc = load().a2ats_select_topk(
        ctypes.byref(shape), ctypes.byref(p), int(n_ctx), _ptr(q, "q", torch.bfloat16),
        _ptr(codes, "codes", _code_dtype(shape)), _ptr(codebook, "codebook", torch.bfloat16),
        _ptr(hist, "hist", torch.int32, optional=True), _ptr(sel_out, "sel_out", torch.int32),
        _ptr(ws, "ws"), ws.numel() * ws.element_size(), _stream(stream))
    _check("a2ats_select_topk", rc)


def a2ats_set_stage_events(events):
    """events: list of >= 5 torch.cuda.Event(enable_timing=True) (already recorded
    once so the handle exists), or None to disable."""
    lib = load()
    if events is None:
        _check("a2ats_set_stage_events", lib.a2ats_set_stage_events(None, 0))
        return
    arr = (ctypes.c_void_p * len(events))(*[e.cuda_event for e in events])
    _check("a2ats_set_stage_events", lib.a2ats_set_stage_events(arr, len(events)))


# ------------------------------------------------------------------ sequence-sharded step
_SZ = ctypes.c_size_t
_SP, _PP = ctypes.POINTER(a2ats_shape), ctypes.POINTER(a2ats_params)
_I32P = ctypes.POINTER(ctypes.c_int32)
_SIGS.update({
    "a2ats_comm_unique_id": (ctypes.c_int, [_VP]),
    "a2ats_comm_init": (ctypes.c_int, [_VP, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_VP)]),
    "a2ats_comm_destroy": (ctypes.c_int, [_VP]),
    "a2ats_shard_state_bytes": (_SZ, [_SP, _PP, ctypes.c_int32]),
    "a2ats_shard_msg_bytes": (_SZ, [_SP]),
    "a2ats_shard_state_layout": (ctypes.c_int, [_SP, _PP, ctypes.c_int32, ctypes.POINTER(_SZ)]),
    "a2ats_shard_workspace_bytes": (_SZ, [_SP, _PP, ctypes.c_int32]),
    "a2ats_shard_state_build": (ctypes.c_int, [_SP, _PP, ctypes.c_int32, ctypes.c_int32, _I32P, ctypes.c_int32, _VP,
                                               _VP, _VP, _SZ, _VP, _VP]),
    "a2ats_decode_step_sharded": (ctypes.c_int, [_SP, _PP, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _I32P,
                                                 _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _SZ, _VP,
                                                 _VP]),
    "a2ats_shard_step_partial": (ctypes.c_int, [_SP, _PP, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _I32P,
                                                _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _SZ, _VP]),
    "a2ats_shard_step_finish": (ctypes.c_int, [_SP, _PP, ctypes.c_int32, ctypes.c_int32, _I32P, _VP, _VP, _VP, _VP]),
    "a2ats_combine": (ctypes.c_int, [_SP, ctypes.c_int32, _VP, _VP, _VP]),
})
if _lib is not None:  # declared after load(): attach the new signatures
    for _n in ("a2ats_comm_unique_id", "a2ats_comm_init", "a2ats_comm_destroy", "a2ats_shard_state_bytes",
               "a2ats_shard_msg_bytes", "a2ats_shard_state_layout", "a2ats_shard_workspace_bytes", "a2ats_shard_state_build",
               "a2ats_decode_step_sharded", "a2ats_shard_step_partial", "a2ats_shard_step_finish", "a2ats_combine"):
        _f = getattr(_lib, _n)
        _f.restype, _f.argtypes = _SIGS[_n]

A2ATS_COMM_ID_BYTES = 128


def _bounds(bounds):
    arr = (ctypes.c_int32 * len(bounds))(*[int(b) for b in bounds])
    return arr


def a2ats_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(A2ATS_COMM_ID_BYTES)
    _check("a2ats_comm_unique_id", load().a2ats_comm_unique_id(buf))
    return buf.raw


def a2ats_comm_init(uid: bytes, world: int, rank: int):
    if len(uid) != A2ATS_COMM_ID_BYTES:
        raise ValueError("uid must be 128 bytes")
    out = _VP()
    buf = ctypes.create_string_buffer(uid, A2ATS_COMM_ID_BYTES)
    _check("a2ats_comm_init", load().a2ats_comm_init(buf, int(world), int(rank), ctypes.byref(out)))
    return out


def a2ats_comm_destroy(comm):
    _check("a2ats_comm_destroy", load().a2ats_comm_destroy(comm))


def a2ats_shard_state_bytes(shape, params, world: int) -> int:
    p = params.c() if isinstance(params, Params) else params
    return int(load().a2ats_shard_state_bytes(ctypes.byref(shape), ctypes.byref(p), int(world)))


def a2ats_shard_state_layout(shape, params, world: int) -> dict:
    p = params.c() if isinstance(params, Params) else params
    off = (_SZ * 6)()
    _check("a2ats_shard_state_layout", load().a2ats_shard_state_layout(ctypes.byref(shape), ctypes.byref(p),
                                                                       int(world), off))
    return dict(hist_g=off[0], hist_r=off[1], ring=off[2], sinkc=off[3], WR=off[4], n_sink_cap=off[5])


def a2ats_shard_msg_bytes(shape) -> int:
    return int(load().a2ats_shard_msg_bytes(ctypes.byref(shape)))


def a2ats_shard_workspace_bytes(shape, params, world: int) -> int:
    p = params.c() if isinstance(params, Params) else params
    return int(load().a2ats_shard_workspace_bytes(ctypes.byref(shape), ctypes.byref(p), int(world)))


def a2ats_shard_state_build(shape, params, world, rank, bounds, n_tokens, codes, state, ws, comm=None, stream=None):
    import torch
    p = params.c() if isinstance(params, Params) else params
    rc = load().a2ats_shard_state_build(ctypes.byref(shape), ctypes.byref(p), int(world), int(rank), _bounds(bounds),
                                        int(n_tokens), _ptr(codes, "codes", _code_dtype(shape)), _ptr(state, "state"),
                                        _ptr(ws, "ws"), ws.numel() * ws.element_size(), comm, _stream(stream))
    _check("a2ats_shard_state_build", rc)


def a2ats_decode_step_sharded(shape, params, n_ctx, world, rank, bounds, q, k_cache, v_cache, codes, codebook, chat,
                              nrm, state, out, sel_out, ws, comm=None, stream=None):
    import torch
    p = params.c() if isinstance(params, Params) else params
    rc = load().a2ats_decode_step_sharded(
        ctypes.byref(shape), ctypes.byref(p), int(n_ctx), int(world), int(rank), _bounds(bounds),
        _ptr(q, "q", torch.bfloat16), _ptr(k_cache, "k_cache", torch.bfloat16), _ptr(v_cache, "v_cache", torch.bfloat16),
        _ptr(codes, "codes", _code_dtype(shape)), _ptr(codebook, "codebook", torch.bfloat16), _ptr(chat, "chat", torch.bfloat16),
        _ptr(nrm, "nrm", torch.float32), _ptr(state, "state"), _ptr(out, "out", torch.float32, host_ok="pinned"),
        _ptr(sel_out, "sel_out", torch.int32, optional=True), _ptr(ws, "ws"), ws.numel() * ws.element_size(), comm,
        _stream(stream))
    _check("a2ats_decode_step_sharded", rc)


def a2ats_shard_step_partial(shape, params, n_ctx, world, rank, bounds, q, k_cache, v_cache, codes, codebook, chat,
                             nrm, state, msg, sel_out, ws, stream=None):
    import torch
    p = params.c() if isinstance(params, Params) else params
    rc = load().a2ats_shard_step_partial(
        ctypes.byref(shape), ctypes.byref(p), int(n_ctx), int(world), int(rank), _bounds(bounds),
        _ptr(q, "q", torch.bfloat16), _ptr(k_cache, "k_cache", torch.bfloat16), _ptr(v_cache, "v_cache", torch.bfloat16),
        _ptr(codes, "codes", _code_dtype(shape)), _ptr(codebook, "codebook", torch.bfloat16), _ptr(chat, "chat", torch.bfloat16),
        _ptr(nrm, "nrm", torch.float32), _ptr(state, "state"), _ptr(msg, "msg"),
        _ptr(sel_out, "sel_out", torch.int32, optional=True), _ptr(ws, "ws"), ws.numel() * ws.element_size(),
        _stream(stream))
    _check("a2ats_shard_step_partial", rc)


def a2ats_shard_step_finish(shape, params, n_ctx, world, bounds, msgs, state, out, stream=None):
    import torch
    p = params.c() if isinstance(params, Params) else params
    rc = load().a2ats_shard_step_finish(ctypes.byref(shape), ctypes.byref(p), int(n_ctx), int(world),
                                        _bounds(bounds), _ptr(msgs, "msgs"), _ptr(state, "state"),
                                        _ptr(out, "out", torch.float32), _stream(stream))
    _check("a2ats_shard_step_finish", rc)


def a2ats_combine(shape, nparts, partials, out, stream=None):
    import torch
    rc = load().a2ats_combine(ctypes.byref(shape), int(nparts), _ptr(partials, "partials", torch.float32),
                              _ptr(out, "out", torch.float32), _stream(stream))
    _check("a2ats_combine", rc)


# ------------------------------------------------------------------ offline codebook construction
_SIGS.update({
    "a2ats_qavq_train_workspace_bytes": (_SZ, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    "a2ats_qavq_train": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _VP, ctypes.c_int32, _VP, _VP,
                                        ctypes.c_double, _VP, ctypes.c_int32, _VP, _VP, _VP, _VP, _VP, _SZ, _VP]),
})
if _lib is not None:
    for _n in ("a2ats_qavq_train_workspace_bytes", "a2ats_qavq_train"):
        _f = getattr(_lib, _n)
        _f.restype, _f.argtypes = _SIGS[_n]


def a2ats_qavq_train_workspace_bytes(n_keys: int, d: int, L: int, m_queries: int = 0) -> int:
    return int(load().a2ats_qavq_train_workspace_bytes(int(n_keys), int(d), int(L), int(m_queries)))


def a2ats_qavq_train(keys, L: int, u, max_iters: int, queries=None, H_in=None, eps: float = 0.0, C_out=None,
                     H_out=None, labels_out=None, info_out=None, ws=None, stream=None):
    """Offline QAVQ codebook of one KV head (device tensors); returns C_out [L, d] fp64."""
    import torch
    n, d = keys.shape
    m = 0 if queries is None else queries.shape[0]
    dev = keys.device
    if C_out is None:
        C_out = torch.empty((L, d), dtype=torch.float64, device=dev)
    if ws is None:
        ws = torch.empty(a2ats_qavq_train_workspace_bytes(n, d, L, m), dtype=torch.uint8, device=dev)
    rc = load().a2ats_qavq_train(int(n), int(d), int(L), _ptr(keys, "keys", torch.bfloat16), int(m),
                                 _ptr(queries, "queries", torch.bfloat16, optional=True),
                                 _ptr(H_in, "H_in", torch.float64, optional=True), float(eps),
                                 _ptr(u, "u", torch.float64), int(max_iters), _ptr(C_out, "C_out", torch.float64),
                                 _ptr(H_out, "H_out", torch.float64, optional=True),
                                 _ptr(labels_out, "labels_out", torch.int32, optional=True),
                                 _ptr(info_out, "info_out", torch.int32, optional=True), _ptr(ws, "ws"),
                                 ws.numel() * ws.element_size(), _stream(stream))
    _check("a2ats_qavq_train", rc)
    return C_out


# ------------------------------------------------------------------ posting-list selection
_SIGS.update({
    "a2ats_postings_bytes": (_SZ, [_SP]),
    "a2ats_postings_build": (ctypes.c_int, [_SP, _VP, ctypes.c_int32, _VP, _VP]),
    "a2ats_select_topk_postings": (ctypes.c_int, [_SP, _PP, ctypes.c_int32, _VP, _VP, _VP, _VP, _VP, ctypes.c_int32,
                                                  _VP, _VP, _SZ, _VP]),
    "a2ats_decode_step_postings": (ctypes.c_int, [_SP, _PP, ctypes.c_int32, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                                  ctypes.c_int32, _VP, _VP, _VP, _SZ, _VP]),
    "a2ats_decode_step_append_postings": (ctypes.c_int, [_SP, _PP, ctypes.c_int32, _VP, _VP, _VP, _VP, _VP, _VP,
                                                         _VP, _VP, _VP, ctypes.c_int32, _VP, _VP, _VP, _SZ, _VP]),
})
if _lib is not None:
    for _n in ("a2ats_postings_bytes", "a2ats_postings_build", "a2ats_select_topk_postings",
               "a2ats_decode_step_postings", "a2ats_decode_step_append_postings"):
        _f = getattr(_lib, _n)
        _f.restype, _f.argtypes = _SIGS[_n]


def a2ats_postings_bytes(shape) -> int:
    return int(load().a2ats_postings_bytes(ctypes.byref(shape)))


def a2ats_postings_build(shape, codes, n_tokens: int, postings, stream=None):
    import torch
    _check("a2ats_postings_build", load().a2ats_postings_build(
        ctypes.byref(shape), _ptr(codes, "codes", _code_dtype(shape)), int(n_tokens), _ptr(postings, "postings"),
        _stream(stream)))


def a2ats_select_topk_postings(shape, params, n_ctx, q, codes, codebook, hist, postings, n_post, sel_out, ws,
                               stream=None):
    import torch
    p = params.c() if isinstance(params, Params) else params
    rc = load().a2ats_select_topk_postings(
        ctypes.byref(shape), ctypes.byref(p), int(n_ctx), _ptr(q, "q", torch.bfloat16), _ptr(codes, "codes", _code_dtype(shape)),
        _ptr(codebook, "codebook", torch.bfloat16), _ptr(hist, "hist", torch.int32), _ptr(postings, "postings"),
        int(n_post), _ptr(sel_out, "sel_out", torch.int32), _ptr(ws, "ws"), ws.numel() * ws.element_size(),
        _stream(stream))
    _check("a2ats_select_topk_postings", rc)


def a2ats_decode_step_postings(shape, params, n_ctx, q, k_cache, v_cache, codes, codebook, hist, postings, n_post,
                               out, sel_out, ws, stream=None):
    import torch
    p = params.c() if isinstance(params, Params) else params
    rc = load().a2ats_decode_step_postings(
        ctypes.byref(shape), ctypes.byref(p), int(n_ctx), _ptr(q, "q", torch.bfloat16),
        _ptr(k_cache, "k_cache", torch.bfloat16), _ptr(v_cache, "v_cache", torch.bfloat16),
        _ptr(codes, "codes", _code_dtype(shape)), _ptr(codebook, "codebook", torch.bfloat16), _ptr(hist, "hist", torch.int32),
        _ptr(postings, "postings"), int(n_post), _ptr(out, "out", torch.float32, host_ok="pinned"),
        _ptr(sel_out, "sel_out", torch.int32, optional=True), _ptr(ws, "ws"), ws.numel() * ws.element_size(),
        _stream(stream))
    _check("a2ats_decode_step_postings", rc)


def a2ats_decode_step_append_postings(shape, params, n_ctx, q, k_cache, v_cache, codes, codebook, hist, chat, nrm,
                                      postings, n_post, out, sel_out, ws, stream=None):
    import torch
    p = params.c() if isinstance(params, Params) else params
    rc = load().a2ats_decode_step_append_postings(
        ctypes.byref(shape), ctypes.byref(p), int(n_ctx), _ptr(q, "q", torch.bfloat16),
        _ptr(k_cache, "k_cache", torch.bfloat16), _ptr(v_cache, "v_cache", torch.bfloat16),
        _ptr(codes, "codes", _code_dtype(shape)), _ptr(codebook, "codebook", torch.bfloat16), _ptr(hist, "hist", torch.int32),
        _ptr(chat, "chat", torch.bfloat16), _ptr(nrm, "nrm", torch.float32), _ptr(postings, "postings"),
        int(n_post), _ptr(out, "out", torch.float32, host_ok="pinned"),
        _ptr(sel_out, "sel_out", torch.int32, optional=True), _ptr(ws, "ws"), ws.numel() * ws.element_size(),
        _stream(stream))
    _check("a2ats_decode_step_append_postings", rc)
