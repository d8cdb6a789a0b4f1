"""Thin ctypes binding of libpariskv.so (include/pariskv.h). Argument marshalling only: every step of the
hot path runs in the library's CUDA kernels; torch supplies device memory and streams. There is no CPU
fallback — importing this module fails loudly when the shared library is missing."""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, f"libpariskv_{os.environ['PKV_LIB']}.so" if os.environ.get("PKV_LIB") else "libpariskv.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libpariskv.so not built ({LIB_PATH}); run `python -m paper_2602_07721_b200.build`")
_lib = ctypes.CDLL(LIB_PATH)

PKV_OK, PKV_ERR_INVALID_ARG, PKV_ERR_CAPACITY, PKV_ERR_CUDA, PKV_ERR_UNSUPPORTED, PKV_ERR_NCCL = 0, -1, -2, -3, -4, -5
D = 128


class PkvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"pariskv status {status}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("head_dim", ctypes.c_int32), ("n_subspaces", ctypes.c_int32), ("subspace_dim", ctypes.c_int32),
                ("n_q_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32), ("n_tiers", ctypes.c_int32),
                ("tier_bonus", ctypes.c_int32 * 8), ("mag_levels", ctypes.c_float * 8),
                ("mag_mid_sq", ctypes.c_double * 7), ("rot_sign", ctypes.c_uint8 * 128),
                ("rot_rounds", ctypes.c_int32), ("w_fp16", ctypes.c_int32)]


class StreamConfig(ctypes.Structure):
    _fields_ = [("sink", ctypes.c_int32), ("local_size", ctypes.c_int32), ("update_size", ctypes.c_int32),
                ("offload_host", ctypes.c_int32)]


class RetrieveParams(ctypes.Structure):
    _fields_ = [("probes_T", ctypes.c_int32), ("n_cand", ctypes.c_int64), ("top_k", ctypes.c_int32),
                ("dbg_scores", ctypes.c_void_p), ("dbg_cand", ctypes.c_void_p), ("dbg_est", ctypes.c_void_p),
                ("dbg_q_rot", ctypes.c_void_p), ("n_global", ctypes.c_int64), ("rho_keys", ctypes.c_int64)]


class IndexStats(ctypes.Structure):
    _fields_ = [("n_keys", ctypes.c_int64), ("zero_keys", ctypes.c_int64),
                ("keys_with_zero_subspace", ctypes.c_int64), ("zero_subspaces", ctypes.c_int64)]


# int32 fn(void* ctx, void* host_buf, size_t bytes_per_rank, int32 rank, int32 world)
HostAllgatherFn = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32,
                                   ctypes.c_int32)


_vp, _i32, _i64, _f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
_sigs = {
    "pkv_config_init": [ctypes.POINTER(Config), _i32, _i32, _vp],
    "pkv_schedule": [_i64, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i64)],
    "pkv_index_create": [ctypes.POINTER(Config), _i32, _i64, _i32, ctypes.POINTER(_vp)],
    "pkv_index_destroy": [_vp],
    "pkv_index_len": [_vp, ctypes.POINTER(_i64)],
    "pkv_index_share_workspace": [_vp, _vp],
    "pkv_index_set_postings": [_vp, _i32, _vp],
    "pkv_index_set_occupancy": [_vp, _i32, _vp],
    "pkv_comm_init_peer": [_vp, _i32, _i32, _i64, ctypes.c_size_t, _vp, ctypes.POINTER(_vp)],
    "pkv_comm_peer_connect": [_vp, _vp],
    "pkv_comm_peer_connect_local": [_vp, _vp],
    "pkv_schedule_key_fraction": [_i64, ctypes.POINTER(_i64)],
    "encode_keys": [_vp, _vp, _i64, _i64, _i64, _i64, _vp],
    "append_decode_keys": [_vp, _vp, _i64, _i64, _i64, _i64, _vp],
    "retrieve_topk": [_vp, _vp, ctypes.POINTER(RetrieveParams), _vp, _vp, _vp],
    "sparse_attend": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _i32, _vp, _vp, _i32, _f32, _vp, _vp, _vp],
    "retrieve_and_attend": [_vp, _vp, ctypes.POINTER(RetrieveParams), _vp, _vp, _i64, _i64, _i64, _vp, _vp, _i32, _f32,
                            _vp, _vp, _vp, _vp, _vp],
    "retrieve_and_attend_rows": [_vp, _vp, ctypes.POINTER(RetrieveParams), _vp, _vp, _i64, _i64, _i64, _vp, _vp,
                                 _i32, _i32, _f32, _vp, _vp, _vp, _vp, _vp],
    "pkv_stream_create": [_vp, ctypes.POINTER(StreamConfig), ctypes.POINTER(_vp)],
    "pkv_stream_destroy": [_vp],
    "pkv_stream_prefill": [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp],
    "pkv_stream_decode": [_vp, _vp, _vp, _vp, ctypes.POINTER(RetrieveParams), _f32, _vp, _vp, _vp, _vp, _vp],
    "pkv_stream_state": [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                         ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp)],
    "pkv_index_export": [_vp, _i64, _i64, _vp, _vp, _vp, _vp],
    "pkv_index_entry_bytes": [_vp, ctypes.POINTER(_i64)],
    "pkv_index_export_front": [_vp, _i64, _vp, _vp],
    "pkv_index_import_back": [_vp, _vp, _i64, _vp],
    "pkv_index_drop_front": [_vp, _i64, _vp],
    "pkv_index_shift_boundary": [_vp, _vp, _i64, _vp],
    "pkv_rebalance_plan": [ctypes.POINTER(_i64), _i32, _i64, ctypes.POINTER(_i64)],
    "pkv_index_get_stats": [_vp, ctypes.POINTER(IndexStats), _vp],
    "pkv_index_set_debug_output": [_vp, _vp],
    "pkv_comm_init_host": [_vp, HostAllgatherFn, _vp, _i32, _i32, _i64],
    "pkv_comm_set_global_len": [_vp, _i64],
    "pkv_nccl_unique_id": [_vp],
    "pkv_comm_init": [_vp, _vp, _i32, _i32, _i64],
    "pkv_comm_share": [_vp, _vp, _i64],
    "pkv_retrieve_topk_sharded_local": [_vp, _vp, _i32, _vp, ctypes.POINTER(RetrieveParams), _vp, _vp, _vp],
    "pkv_sparse_attend_sharded_local": [_vp, _vp, _i32, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _i32, _vp, _vp, _i32,
                                        _f32, _vp, _vp, _vp],
    "pkv_retrieve_and_attend_sharded_local": [_vp, _vp, _i32, _vp, _vp, _vp, _i64, _i64, _i64,
                                              ctypes.POINTER(RetrieveParams), _vp, _vp, _i32, _f32, _vp, _vp, _vp,
                                              _vp, _vp],
    "pkv_launch_count": [ctypes.POINTER(ctypes.c_uint64)],
    "pkv_profile_enable": [_i32],
    "pkv_profile_read": [_i32, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_double)],
}
for _name, _args in _sigs.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = ctypes.c_int
_lib.pkv_last_error.restype = ctypes.c_char_p
_lib.pkv_version.restype = ctypes.c_char_p
_lib.pkv_kernel_name.restype = ctypes.c_char_p
_lib.pkv_kernel_name.argtypes = [_i32]

EXPORTED = tuple(_sigs) + ("pkv_last_error", "pkv_version", "pkv_kernel_name")
KERNEL_KINDS = ("encode", "qprep", "scan", "select", "unused", "rerank", "topk", "topk_merge", "attend",
                "combine", "head_hist", "export", "debug")


def _check(status: int):
    if status != PKV_OK:
        raise PkvError(status, _lib.pkv_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def version() -> str:
    return _lib.pkv_version().decode()


def launch_count() -> int:
    v = ctypes.c_uint64(0)
    _check(_lib.pkv_launch_count(ctypes.byref(v)))
    return int(v.value)


def profile_enable(on: bool):
    _check(_lib.pkv_profile_enable(1 if on else 0))


def profile_read() -> dict:
    """{kernel kind: (launches, total device ms)} since the last profile_enable."""
    out = {}
    for i, name in enumerate(KERNEL_KINDS):
        n, ms = _i64(0), ctypes.c_double(0)
        _check(_lib.pkv_profile_read(i, ctypes.byref(n), ctypes.byref(ms)))
        if n.value:
            out[name] = (int(n.value), float(ms.value))
    return out


def config_init(n_q_heads: int, n_kv_heads: int, rot_sign_bits) -> Config:
    cfg = Config()
    signs = np.ascontiguousarray(np.asarray(rot_sign_bits, dtype=np.uint8))
    assert signs.shape == (D,)
    _check(_lib.pkv_config_init(ctypes.byref(cfg), n_q_heads, n_kv_heads, signs.ctypes.data_as(ctypes.c_void_p)))
    return cfg


def schedule(n: int, top_k: int):
    T, C = _i32(0), _i64(0)
    _check(_lib.pkv_schedule(n, top_k, ctypes.byref(T), ctypes.byref(C)))
    return int(T.value), int(C.value)


def schedule_key_fraction(n: int) -> int:
    """rho_keys = ceil(rho n) for the key-fraction reading of rho (AMB-8b)."""
    r = _i64(0)
    _check(_lib.pkv_schedule_key_fraction(n, ctypes.byref(r)))
    return int(r.value)


class Index:
    """Owns a pkv_index (GPU-resident key summaries of the retrieval zone)."""

    def __init__(self, cfg: Config, batch: int, capacity: int, device: int = 0):
        self.cfg = cfg
        self.batch = batch
        self.capacity = capacity
        self.device = device
        self.n_q = cfg.n_q_heads
        self.n_kv = cfg.n_kv_heads
        h = _vp()
        _check(_lib.pkv_index_create(ctypes.byref(cfg), batch, capacity, device, ctypes.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            _lib.pkv_index_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self):
        n = _i64(0)
        _check(_lib.pkv_index_len(self.handle, ctypes.byref(n)))
        return int(n.value)

    def set_postings(self, enable: bool = True, stream=None):
        """Inverted-list collision variant: same results, buckets of probed centroids only."""
        _check(_lib.pkv_index_set_postings(self.handle, int(enable), _stream(stream)))

    def comm_init_peer(self, rank: int, world: int, shard_offset: int, arena_bytes: int = 64 << 20):
        """Peer transport: allocate this rank's exchange arena; returns (ipc_handle bytes, arena ptr)."""
        h = (ctypes.c_uint8 * 64)()
        a = _vp()
        _check(_lib.pkv_comm_init_peer(self.handle, rank, world, shard_offset, arena_bytes, h, ctypes.byref(a)))
        return bytes(h), int(a.value)

    def comm_peer_connect(self, handles):
        """Open the peers' arenas from their IPC handles (list of `world` 64-byte strings, ranks in other processes)."""
        buf = (ctypes.c_uint8 * (64 * len(handles))).from_buffer_copy(b"".join(handles))
        _check(_lib.pkv_comm_peer_connect(self.handle, buf))

    def comm_peer_connect_local(self, arenas):
        """Connect to the other ranks' arenas by device pointer (ranks in this process)."""
        arr = (ctypes.c_void_p * len(arenas))(*arenas)
        _check(_lib.pkv_comm_peer_connect_local(self.handle, arr))

    def set_occupancy(self, enable: bool = True, stream=None):
        """Per-subspace centroid occupancy counts, needed by retrievals with rho_keys > 0 (AMB-8b)."""
        _check(_lib.pkv_index_set_occupancy(self.handle, int(enable), _stream(stream)))

    def stats(self, stream=None) -> dict:
        """Degenerate-key counters of the current content (AMB-7; synchronises the stream)."""
        s = IndexStats()
        _check(_lib.pkv_index_get_stats(self.handle, ctypes.byref(s), _stream(stream)))
        return {f: int(getattr(s, f)) for f, _ in IndexStats._fields_}

    def set_debug_output(self, out_f32: torch.Tensor | None):
        """fp32 copy [batch, n_q, 128] of every later attention output on this index (None disables)."""
        if out_f32 is not None:
            assert out_f32.dtype == torch.float32 and out_f32.is_contiguous()
            assert tuple(out_f32.shape) == (self.batch, self.n_q, D)
        self._dbg_out = out_f32  # kept alive while the library holds the pointer
        _check(_lib.pkv_index_set_debug_output(self.handle, _ptr(out_f32)))

    def share_workspace(self, donor: "Index"):
        _check(_lib.pkv_index_share_workspace(self.handle, donor.handle))

    def export(self, start: int = 0, count: int | None = None, stream=None):
        """Canonical metadata of positions [start, start+count): (ids u8 [b,kv,c,16], codes u8 [b,kv,c,64],
        w f32 [b,kv,c,16])."""
        count = len(self) - start if count is None else count
        dev = torch.device("cuda", self.device)
        ids = torch.empty(self.batch, self.n_kv, count, 16, dtype=torch.uint8, device=dev)
        codes = torch.empty(self.batch, self.n_kv, count, 64, dtype=torch.uint8, device=dev)
        w = torch.empty(self.batch, self.n_kv, count, 16, dtype=torch.float32, device=dev)
        _check(_lib.pkv_index_export(self.handle, start, count, _ptr(ids), _ptr(codes), _ptr(w), _stream(stream)))
        return ids, codes, w


    # ---- append rebalancing across sequence shards (pkv_index_export_front / import_back / drop_front)
    def entry_bytes(self) -> int:
        v = _i64(0)
        _check(_lib.pkv_index_entry_bytes(self.handle, ctypes.byref(v)))
        return int(v.value)

    def export_front(self, count: int, stream=None) -> torch.Tensor:
        """Entries of the `count` oldest keys, u8 [count * entry_bytes] on the index's device."""
        buf = torch.empty(max(1, count * self.entry_bytes()), dtype=torch.uint8, device=torch.device("cuda", self.device))
        _check(_lib.pkv_index_export_front(self.handle, count, _ptr(buf), _stream(stream)))
        return buf

    def import_back(self, buf: torch.Tensor, count: int, stream=None):
        assert buf.dtype == torch.uint8 and buf.is_contiguous() and buf.numel() >= count * self.entry_bytes()
        _check(_lib.pkv_index_import_back(self.handle, _ptr(buf), count, _stream(stream)))

    def drop_front(self, count: int, stream=None):
        _check(_lib.pkv_index_drop_front(self.handle, count, _stream(stream)))


def shift_boundary(older: Index, newer: Index, count: int, stream=None):
    """Move the `count` oldest keys of `newer` to the end of `older` (same device)."""
    _check(_lib.pkv_index_shift_boundary(older.handle, newer.handle, count, _stream(stream)))


def rebalance_plan(lengths, granule: int = 512) -> list:
    """shift[r] = keys to move from shard r+1 to shard r (apply from the last boundary to the first)."""
    P = len(lengths)
    arr = (_i64 * P)(*[int(x) for x in lengths])
    out = (_i64 * max(1, P - 1))()
    _check(_lib.pkv_rebalance_plan(arr, P, granule, out))
    return [int(out[i]) for i in range(P - 1)]


def _kv_strides(K: torch.Tensor):
    assert K.dtype == torch.bfloat16 and K.dim() == 4 and K.shape[-1] == D and K.stride(-1) == 1
    return K.stride(0), K.stride(1), K.stride(2)


def encode_keys(index: Index, K: torch.Tensor, n: int | None = None, stream=None):
    """(1) prefill: K bf16 [batch, n_kv, tokens, 128] (any strides with unit last stride)."""
    n = K.shape[2] if n is None else n
    sb, sh, st = _kv_strides(K)
    _check(_lib.encode_keys(index.handle, _ptr(K), sb, sh, st, n, _stream(stream)))


def append_decode_keys(index: Index, K: torch.Tensor, t: int | None = None, stream=None):
    """(2) decode flush: append the t keys of K bf16 [batch, n_kv, t, 128]."""
    t = K.shape[2] if t is None else t
    sb, sh, st = _kv_strides(K)
    _check(_lib.append_decode_keys(index.handle, _ptr(K), sb, sh, st, t, _stream(stream)))


def retrieve_topk(index: Index, q: torch.Tensor, top_k: int, probes_T: int | None = None, n_cand: int | None = None,
                  n_global: int | None = None, out_idx=None, out_est=None, debug: bool = False, rho_keys: int = 0,
                  stream=None):
    """(3) q bf16 [batch, n_q, 128] -> (idx int32 [batch, n_q, k], est f32 [batch, n_q, k], dbg dict|None).
    probes_T / n_cand default to the library schedule on the (global) retrieval length."""
    assert q.dtype == torch.bfloat16 and q.is_contiguous() and q.shape[-1] == D
    n = len(index) if n_global is None else n_global
    T0, C0 = schedule(n, top_k)
    T = T0 if probes_T is None else probes_T
    C = C0 if n_cand is None else n_cand
    dev = q.device
    if out_idx is None:
        out_idx = torch.empty(index.batch, index.n_q, top_k, dtype=torch.int32, device=dev)
    if out_est is None:
        out_est = torch.empty(index.batch, index.n_q, top_k, dtype=torch.float32, device=dev)
    p = RetrieveParams(T, C, top_k, None, None, None, None, 0 if n_global is None else n_global, rho_keys)
    dbg = None
    if debug:
        nl = len(index)
        dbg = dict(scores=torch.empty(index.batch, index.n_q, nl, dtype=torch.uint8, device=dev),
                   cand=torch.empty(index.batch, index.n_q, C, dtype=torch.int32, device=dev),
                   est=torch.empty(index.batch, index.n_q, C, dtype=torch.float32, device=dev),
                   q_rot=torch.empty(index.batch, index.n_q, D, dtype=torch.float32, device=dev), T=T, C=C)
        p.dbg_scores, p.dbg_cand = dbg["scores"].data_ptr(), dbg["cand"].data_ptr()
        p.dbg_est, p.dbg_q_rot = dbg["est"].data_ptr(), dbg["q_rot"].data_ptr()
    _check(_lib.retrieve_topk(index.handle, _ptr(q), ctypes.byref(p), _ptr(out_idx), _ptr(out_est), _stream(stream)))
    return out_idx, out_est, dbg


def sparse_attend(index: Index, q: torch.Tensor, K: torch.Tensor | None, V: torch.Tensor | None, idx, K_hot=None,
                  V_hot=None, scale: float | None = None, out=None, lse=None, strides=None, K_ptr=None, V_ptr=None,
                  stream=None):
    """(4) attention over hot rows U retrieved rows. K/V: bf16 [batch, n_kv, tokens, 128] device tensors, or pass
    raw UVA pointers K_ptr/V_ptr (int) with `strides` (sb, sh, st) for pinned host memory."""
    k = 0 if idx is None else idx.shape[-1]
    n_hot = 0 if K_hot is None else K_hot.shape[2]
    scale = 1.0 / np.sqrt(D) if scale is None else scale
    if K_ptr is None:
        if K is not None:
            sb, sh, st = _kv_strides(K)
            assert V.stride() == K.stride()
            K_ptr, V_ptr = K.data_ptr(), V.data_ptr()
        else:
            sb = sh = st = 0
            K_ptr = V_ptr = None
    else:
        sb, sh, st = strides
    if out is None:
        out = torch.empty(index.batch, index.n_q, D, dtype=torch.bfloat16, device=q.device)
    if lse is None:
        lse = torch.empty(index.batch, index.n_q, dtype=torch.float32, device=q.device)
    if K_hot is not None:
        assert K_hot.is_contiguous() and V_hot.is_contiguous()
    _check(_lib.sparse_attend(index.handle, _ptr(q), _vp(K_ptr), _vp(V_ptr), sb, sh, st, _ptr(idx), k,
                              _ptr(K_hot), _ptr(V_hot), n_hot, scale, _ptr(out), _ptr(lse), _stream(stream)))
    return out, lse


def retrieve_and_attend(index: Index, q: torch.Tensor, K, V, top_k: int, K_hot=None, V_hot=None,
                        scale: float | None = None, probes_T: int | None = None, n_cand: int | None = None,
                        out_idx=None, out_est=None, out=None, lse=None, strides=None, K_ptr=None, V_ptr=None,
                        n_global: int | None = None, rho_keys: int = 0, stream=None):
    """(3)+(4) in one call: retrieval and attention of one decode step and layer, with the hot-row attention
    overlapped with the retrieval and the final top-k fused with the gather/attention. Returns
    (idx, est, out, lse)."""
    assert q.dtype == torch.bfloat16 and q.is_contiguous() and q.shape[-1] == D
    n = len(index) if n_global is None else n_global
    T0, C0 = schedule(n, top_k)
    T = T0 if probes_T is None else probes_T
    C = C0 if n_cand is None else n_cand
    dev = q.device
    if out_idx is None:
        out_idx = torch.empty(index.batch, index.n_q, top_k, dtype=torch.int32, device=dev)
    if out_est is None:
        out_est = torch.empty(index.batch, index.n_q, top_k, dtype=torch.float32, device=dev)
    if out is None:
        out = torch.empty(index.batch, index.n_q, D, dtype=torch.bfloat16, device=dev)
    if lse is None:
        lse = torch.empty(index.batch, index.n_q, dtype=torch.float32, device=dev)
    if K_ptr is None:
        sb, sh, st = _kv_strides(K)
        K_ptr, V_ptr = K.data_ptr(), V.data_ptr()
    else:
        sb, sh, st = strides
    n_hot = 0 if K_hot is None else K_hot.shape[2]
    scale = 1.0 / np.sqrt(D) if scale is None else scale
    p = RetrieveParams(T, C, top_k, None, None, None, None, 0 if n_global is None else n_global, rho_keys)
    _check(_lib.retrieve_and_attend(index.handle, _ptr(q), ctypes.byref(p), _vp(K_ptr), _vp(V_ptr), sb, sh, st,
                                    _ptr(K_hot), _ptr(V_hot), n_hot, scale, _ptr(out_idx), _ptr(out_est), _ptr(out),
                                    _ptr(lse), _stream(stream)))
    return out_idx, out_est, out, lse


class Stream:
    """Four-region streaming KV cache of one layer (PAPER §4.2.3; include/pariskv.h pkv_stream_*):
    Sink + Local + Update buffer on the GPU, older tokens indexed in `index` with their K/V in a store owned by
    the stream (HBM, or pinned host memory read through UVA when offload_host)."""

    def __init__(self, index: Index, sink: int = 16, local_size: int = 256, update_size: int = 512,
                 offload_host: bool = False):
        self.index = index
        self.cfg = StreamConfig(sink, local_size, update_size, int(offload_host))
        h = _vp()
        _check(_lib.pkv_stream_create(index.handle, ctypes.byref(self.cfg), ctypes.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            _lib.pkv_stream_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prefill(self, K: torch.Tensor, V: torch.Tensor, stream=None):
        """K, V bf16 [batch, n_kv, tokens, 128] (unit last stride, same strides)."""
        sb, sh, st = _kv_strides(K)
        assert _kv_strides(V) == (sb, sh, st)
        _check(_lib.pkv_stream_prefill(self.handle, _ptr(K), _ptr(V), sb, sh, st, K.shape[2], _stream(stream)))

    def decode(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, top_k: int, scale=None,
               probes_T: int = 0, n_cand: int = 0, out_idx=None, out_est=None, out=None, lse=None, debug=None,
               stream=None):
        """One decode step: q bf16 [batch, n_q, 128]; k_new, v_new bf16 [batch, n_kv, 128] (contiguous).
        probes_T / n_cand = 0: the schedule for the current retrieval length. Returns (idx, est, out, lse);
        idx are retrieval-store positions (token = sink + idx)."""
        ix = self.index
        dev = q.device
        assert k_new.is_contiguous() and v_new.is_contiguous() and q.is_contiguous()
        if out_idx is None:
            out_idx = torch.empty(ix.batch, ix.n_q, top_k, dtype=torch.int32, device=dev)
        if out_est is None:
            out_est = torch.empty(ix.batch, ix.n_q, top_k, dtype=torch.float32, device=dev)
        if out is None:
            out = torch.empty(ix.batch, ix.n_q, D, dtype=torch.bfloat16, device=dev)
        if lse is None:
            lse = torch.empty(ix.batch, ix.n_q, dtype=torch.float32, device=dev)
        scale = 1.0 / np.sqrt(D) if scale is None else scale
        p = RetrieveParams(probes_T, n_cand, top_k, None, None, None, None)
        if debug is not None:  # dict of preallocated tensors: scores [b,q,n_after], cand/est [b,q,C], q_rot
            p.dbg_scores = debug["scores"].data_ptr() if "scores" in debug else None
            p.dbg_cand = debug["cand"].data_ptr() if "cand" in debug else None
            p.dbg_est = debug["est"].data_ptr() if "est" in debug else None
            p.dbg_q_rot = debug["q_rot"].data_ptr() if "q_rot" in debug else None
        _check(_lib.pkv_stream_decode(self.handle, _ptr(q), _ptr(k_new), _ptr(v_new), ctypes.byref(p), scale,
                                      _ptr(out_idx), _ptr(out_est), _ptr(out), _ptr(lse), _stream(stream)))
        return out_idx, out_est, out, lse

    def state(self):
        """(n_retrieval, n_local, n_buffer)."""
        n = _i64(0)
        nl, nb = _i32(0), _i32(0)
        _check(_lib.pkv_stream_state(self.handle, ctypes.byref(n), ctypes.byref(nl), ctypes.byref(nb), None, None,
                                     None, None))
        return int(n.value), int(nl.value), int(nb.value)

    def views(self):
        """Torch views of the retrieval store (K, V [batch, n_kv, capacity, 128]) and of the hot buffer
        (K, V [batch, n_kv, sink + local_size + update_size, 128]) — for tests and diagnostics."""
        ptrs = [_vp() for _ in range(4)]
        _check(_lib.pkv_stream_state(self.handle, None, None, None, *[ctypes.byref(p) for p in ptrs]))
        ix = self.index
        rows = self.cfg.sink + self.cfg.local_size + self.cfg.update_size
        shapes = [(ix.batch, ix.n_kv, ix.capacity, D)] * 2 + [(ix.batch, ix.n_kv, rows, D)] * 2
        return tuple(_wrap_bf16(p.value, shp, ix.device) for p, shp in zip(ptrs, shapes))


def _wrap_bf16(ptr: int, shape, device: int) -> torch.Tensor:
    """Non-owning torch view of library-owned bf16 device memory (valid while its owner lives)."""
    n = int(np.prod(shape))

    class _Cuda:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (ptr, False), "version": 3}

    with torch.cuda.device(device):
        return torch.as_tensor(_Cuda(), device=f"cuda:{device}").view(torch.bfloat16).view(*shape)


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(_lib.pkv_nccl_unique_id(buf))
    return bytes(buf)


def comm_init(index: Index, uid: bytes, rank: int, world: int, shard_offset: int):
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _check(_lib.pkv_comm_init(index.handle, buf, rank, world, shard_offset))


def comm_init_host(index: Index, allgather, rank: int, world: int, shard_offset: int):
    """Attach the host-staged transport: allgather(buf: numpy uint8 [world, bytes_per_rank]) must fill every row
    with that rank's bytes in place (row `rank` holds this rank's on entry), e.g. a gloo all_gather."""
    def _fn(ctx, buf, nbytes, r, w):
        try:
            arr = np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(ctypes.c_uint8)), shape=(w * nbytes,))
            allgather(arr.reshape(w, nbytes))
            return 0
        except Exception:  # noqa: BLE001 — reported to the library as a failed exchange
            import traceback
            traceback.print_exc()
            return 1
    cb = HostAllgatherFn(_fn)
    index._allgather_cb = cb  # the library keeps the pointer: keep the trampoline alive with the index
    _check(_lib.pkv_comm_init_host(index.handle, cb, None, rank, world, shard_offset))


def comm_set_global_len(index: Index, n_global: int):
    _check(_lib.pkv_comm_set_global_len(index.handle, n_global))


def comm_share(index: Index, donor: Index, shard_offset: int):
    _check(_lib.pkv_comm_share(index.handle, donor.handle, shard_offset))


def retrieve_topk_sharded_local(shards, offsets, q, top_k, n_global, stream=None):
    P = len(shards)
    T, C = schedule(n_global, top_k)
    hs = (_vp * P)(*[s.handle.value for s in shards])
    offs = (_i64 * P)(*offsets)
    out_idx = torch.empty(shards[0].batch, shards[0].n_q, top_k, dtype=torch.int32, device=q.device)
    out_est = torch.empty(shards[0].batch, shards[0].n_q, top_k, dtype=torch.float32, device=q.device)
    p = RetrieveParams(T, C, top_k, None, None, None, None)
    _check(_lib.pkv_retrieve_topk_sharded_local(hs, offs, P, _ptr(q), ctypes.byref(p), _ptr(out_idx), _ptr(out_est),
                                                _stream(stream)))
    return out_idx, out_est


def retrieve_and_attend_sharded_local(shards, offsets, q, Ks, Vs, top_k, K_hot=None, V_hot=None, scale=None,
                                      stream=None):
    """Single-process emulation of the sequence-sharded retrieve_and_attend with the fused exchange (§8(f3)):
    shard p owns global positions [offsets[p], offsets[p] + len(shards[p])); Ks[p], Vs[p] its K/V rows."""
    P = len(shards)
    n_global = sum(len(s) for s in shards)
    T, C = schedule(n_global, top_k)
    hs = (_vp * P)(*[s.handle.value for s in shards])
    offs = (_i64 * P)(*offsets)
    kp = (_vp * P)(*[k.data_ptr() for k in Ks])
    vp = (_vp * P)(*[v.data_ptr() for v in Vs])
    sb, sh, st = _kv_strides(Ks[0])
    ix = shards[0]
    dev = q.device
    out_idx = torch.empty(ix.batch, ix.n_q, top_k, dtype=torch.int32, device=dev)
    out_est = torch.empty(ix.batch, ix.n_q, top_k, dtype=torch.float32, device=dev)
    out = torch.empty(ix.batch, ix.n_q, D, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(ix.batch, ix.n_q, dtype=torch.float32, device=dev)
    n_hot = 0 if K_hot is None else K_hot.shape[2]
    scale = 1.0 / np.sqrt(D) if scale is None else scale
    p = RetrieveParams(T, C, top_k, None, None, None, None)
    _check(_lib.pkv_retrieve_and_attend_sharded_local(hs, offs, P, _ptr(q), kp, vp, sb, sh, st, ctypes.byref(p),
                                                      _ptr(K_hot), _ptr(V_hot), n_hot, scale, _ptr(out_idx),
                                                      _ptr(out_est), _ptr(out), _ptr(lse), _stream(stream)))
    return out_idx, out_est, out, lse


def sparse_attend_sharded_local(shards, offsets, q, Ks, Vs, idx, K_hot=None, V_hot=None, scale=None, stream=None):
    P = len(shards)
    k = idx.shape[-1]
    n_hot = 0 if K_hot is None else K_hot.shape[2]
    scale = 1.0 / np.sqrt(D) if scale is None else scale
    sb, sh, st = _kv_strides(Ks[0])
    hs = (_vp * P)(*[s.handle.value for s in shards])
    offs = (_i64 * P)(*offsets)
    kp = (_vp * P)(*[t.data_ptr() for t in Ks])
    vp = (_vp * P)(*[t.data_ptr() for t in Vs])
    out = torch.empty(shards[0].batch, shards[0].n_q, D, dtype=torch.bfloat16, device=q.device)
    lse = torch.empty(shards[0].batch, shards[0].n_q, dtype=torch.float32, device=q.device)
    _check(_lib.pkv_sparse_attend_sharded_local(hs, offs, P, _ptr(q), kp, vp, sb, sh, st, _ptr(idx), k, _ptr(K_hot),
                                                _ptr(V_hot), n_hot, scale, _ptr(out), _ptr(lse), _stream(stream)))
    return out, lse
