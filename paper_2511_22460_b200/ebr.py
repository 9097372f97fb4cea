"""Thin ctypes binding of include/ebr.h (argument marshalling only).

Every step of the hot path runs in the CUDA library libebr.so; this module only passes pointers
(numpy arrays for host inputs, torch tensors for device buffers, a CUDA stream handle) and turns
status codes into exceptions.  There is no fallback: if libebr.so is missing or fails to load,
importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# EBR_LIB: an alternative build of the same library (A/B measurements); default the in-tree one
LIB_PATH = os.environ.get("EBR_LIB") or os.path.join(_HERE, "libebr.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                      " (there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

F32, BF16 = 0, 1
MAX_K = 16384
STATUS = {0: "EBR_OK", 1: "EBR_EINVAL", 2: "EBR_ENOMEM", 3: "EBR_ECUDA", 4: "EBR_EUNSUPPORTED",
          5: "EBR_EDEVICE"}

_P, _I32, _I64, _SZ, _U32P = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p

EXPORTS = {
    # name: (restype, argtypes)
    "ebr_build_index": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _I32, _P, _I32, _P, _P, _I64,
                                       ctypes.c_int, _P, ctypes.POINTER(_P)]),
    "ebr_build_index_device": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _I32, _P, _I32, _P, _P, _I64,
                                              ctypes.c_int, _P, ctypes.POINTER(_P)]),
    "ebr_build_index_lists": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _I32, _P, _P, _I32, _P, _P, _I64,
                                             ctypes.c_int, _P, ctypes.POINTER(_P)]),
    "ebr_index_export": (ctypes.c_int, [_P, _I32, _P, _I64, ctypes.POINTER(_I64)]),
    "ebr_free_index": (None, [_P]),
    "ebr_workspace_bytes": (_SZ, [_P, _I32, _I32, _I32]),
    "ebr_score_topk": (ctypes.c_int, [_P, _P, _I32, _P, _P, _I32, _I32, _P, _P, _P, _SZ, _P]),
    "ebr_score_topk_keys": (ctypes.c_int, [_P, _P, _I32, _P, _P, _I32, _I32, _P, _P, _SZ, _P]),
    "ebr_query_error": (ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_uint32)]),
    "ebr_workspace_init": (ctypes.c_int, [_P, _P, _SZ, _P]),
    "ebr_workspace_bytes_host": (_SZ, [_P, _I32, _I32, _I32]),
    "ebr_score_topk_host": (ctypes.c_int, [_P, _P, _I32, _P, _P, _I32, _I32, _P, _P, _P, _SZ, _P]),
    "ebr_merge_workspace_bytes": (_SZ, [_I32, _I32, _I32]),
    "ebr_merge_topk": (ctypes.c_int, [_P, _I32, _I32, _I32, _P, _P, _P, _SZ, _P]),
    "ebr_debug_decode": (ctypes.c_int, [_P, _I64, _P, _I64, ctypes.POINTER(_I64)]),
    "ebr_index_stats": (ctypes.c_int, [_P, _P]),
    "ebr_encode_host": (ctypes.c_int, [_P, _I64, _I32, _P, _I64, _P, _P, _P, _I64, _P, _I64,
                                       ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "ebr_query_launches": (_I32, [_P, _I32, _I32, _I32]),
    "ebr_exchange_kth": (ctypes.c_int, [_P, _I32, _I32, _I32, _P, _P]),
    "ebr_exchange_pack": (ctypes.c_int, [_P, _I32, _I32, _P, _I32, _P, _P, _P, _P]),
    "ebr_merge_topk_packed": (ctypes.c_int, [_P, _I64, _P, _I32, _I32, _I32, _P, _P, _P]),
    "ebr_paper_index_build": (ctypes.c_int, [_P, _I64, _I32, _P, _I64, ctypes.c_int, _P, ctypes.POINTER(_P)]),
    "ebr_paper_index_free": (None, [_P]),
    "ebr_paper_index_info": (ctypes.c_int, [_P, _P, ctypes.POINTER(_I64), ctypes.POINTER(ctypes.c_double)]),
    "ebr_paper_hitmatch": (ctypes.c_int, [_P, _P, _P, _I32, _P, _P]),
    "ebr_chunk_hitmatch": (ctypes.c_int, [_P, _P, _P, _I32, _P, _P]),
    "ebr_ipnn_extend": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _I32, ctypes.c_int, _P, _P]),
    "ebr_kernel_timer": (ctypes.c_int, [_I32]),
    "ebr_kernel_timer_read": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64),
                                             ctypes.c_char_p, _I32]),
    "ebr_last_error": (ctypes.c_char_p, []),
    "ebr_version": (ctypes.c_char_p, []),
}
for _name, (_res, _args) in EXPORTS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class EbrError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}: {last_error()}")


def last_error() -> str:
    return _lib.ebr_last_error().decode()


def version() -> str:
    return _lib.ebr_version().decode()


class PaperIndex:
    """NEXT-3 ablation: the paper's own inverted list (Alg. 1) on the GPU (ebr_paper_index_build)."""

    def __init__(self, ad_feat, field_card, device: int = 0, stream=None):
        ad_feat = np.ascontiguousarray(ad_feat, np.int32)
        field_card = np.ascontiguousarray(field_card, np.int32)
        self.n_ads, self.n_fields = ad_feat.shape
        self.n_keys = int(field_card.astype(np.int64).sum())
        h = ctypes.c_void_p()
        _check(_lib.ebr_paper_index_build(_np_ptr(ad_feat), self.n_ads, self.n_fields, _np_ptr(field_card),
                                          self.n_keys, device, _stream_ptr(stream), ctypes.byref(h)),
               "ebr_paper_index_build")
        self._h = h

    def info(self) -> dict:
        blocks = np.zeros(9, np.int64)
        nb, ms = ctypes.c_int64(0), ctypes.c_double(0.0)
        _check(_lib.ebr_paper_index_info(self._h, _np_ptr(blocks), ctypes.byref(nb), ctypes.byref(ms)),
               "ebr_paper_index_info")
        return {"blocks_per_group": blocks.tolist(), "bytes": nb.value, "build_ms": ms.value}

    def close(self):
        if getattr(self, "_h", None):
            _lib.ebr_paper_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def paper_hitmatch(pidx: PaperIndex, keys, w, scores, stream=None):
    """Alg. 2 on the paper's layout: scores[a] = sum_i w[i] L[a, keys[i]] (device tensors)."""
    _check(_lib.ebr_paper_hitmatch(pidx._h, _t_ptr(keys), _t_ptr(w), keys.shape[0], _t_ptr(scores),
                                   _stream_ptr(stream)), "ebr_paper_hitmatch")


def chunk_hitmatch(idx: Index, keys, w, scores, stream=None):
    """The same algorithm on this library's chunk codec (ebr_chunk_hitmatch)."""
    _check(_lib.ebr_chunk_hitmatch(idx.handle, _t_ptr(keys), _t_ptr(w), keys.shape[0], _t_ptr(scores),
                                   _stream_ptr(stream)), "ebr_chunk_hitmatch")


def ipnn_extend(h, u, W, out, stream=None):
    """h~ = [h, W u] per row (Eq. 7-8) on the device: h [rows][d0] float32 or int16 (bf16 bits),
    u [rows][n] float32, W [d1][n] float32, out [rows][d0 + d1] in h's dtype."""
    rows, d0 = h.shape
    d1, n = W.shape
    dtype = BF16 if h.element_size() == 2 else F32
    _check(_lib.ebr_ipnn_extend(_t_ptr(h), _t_ptr(u), _t_ptr(W), rows, d0, n, d1, dtype, _t_ptr(out),
                                _stream_ptr(stream)), "ebr_ipnn_extend")


def kernel_timer(enable: bool) -> None:
    """Start/stop recording CUDA events around each query's dominant kernel (ebr.h)."""
    _check(_lib.ebr_kernel_timer(1 if enable else 0), "ebr_kernel_timer")


def kernel_timer_read() -> tuple[float, int, str]:
    """(summed ms, timed launches, kernel name) of the recorded launches; clears the record."""
    ms, n = ctypes.c_double(0.0), ctypes.c_int64(0)
    name = ctypes.create_string_buffer(256)
    _check(_lib.ebr_kernel_timer_read(ctypes.byref(ms), ctypes.byref(n), name, 256), "ebr_kernel_timer_read")
    return ms.value, n.value, name.value.decode()


def _check(st: int, where: str):
    if st != 0:
        raise EbrError(st, where)


class Stats(ctypes.Structure):
    _fields_ = [("n_ads", _I64), ("ad_begin", _I64), ("d", _I32), ("d_pad", _I32),
                ("dtype", _I32), ("n_fields", _I32), ("n_keys", _I64), ("nnz", _I64),
                ("chunks", _I64), ("payload_words", _I64), ("index_bytes", _I64),
                ("emb_bytes", _I64), ("build_ms", ctypes.c_double), ("n_hot", _I32),
                ("pad0", _I32), ("hot_nnz", _I64), ("hot_bytes", _I64), ("encode_ms", ctypes.c_double)]


def _np_ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _t_ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    if stream is None:
        return None
    return ctypes.c_void_p(int(getattr(stream, "cuda_stream", stream)))


class Index:
    """An inventory shard resident on one GPU (ebr_build_index / ebr_free_index)."""

    def __init__(self, ad_emb, ad_feat, field_card, cross_w, ad_begin: int = 0, device: int = 0,
                 stream=None, device_build: bool = False):
        ad_emb = np.ascontiguousarray(ad_emb)
        if ad_emb.dtype == np.uint16:
            self.dtype = BF16
        elif ad_emb.dtype == np.float32:
            self.dtype = F32
        else:
            raise TypeError("ad_emb must be float32 or uint16 (bf16 bits)")
        ad_feat = np.ascontiguousarray(ad_feat, np.int32)
        field_card = np.ascontiguousarray(field_card, np.int32)
        cross_w = np.ascontiguousarray(cross_w, np.float32)
        n, self.d = ad_emb.shape
        self.n_fields = field_card.shape[0]
        self.n_keys = int(field_card.astype(np.int64).sum())
        self.ad_begin = int(ad_begin)
        self.n_ads = int(n)
        self.device = device
        h = ctypes.c_void_p()
        fn = _lib.ebr_build_index_device if device_build else _lib.ebr_build_index
        st = fn(_np_ptr(ad_emb), self.dtype, self.ad_begin, self.ad_begin + n,
                                  self.d, _np_ptr(ad_feat), self.n_fields, _np_ptr(field_card),
                                  _np_ptr(cross_w), self.n_keys, device, _stream_ptr(stream),
                                  ctypes.byref(h))
        _check(st, "ebr_build_index_device" if device_build else "ebr_build_index")
        self._h = h

    @classmethod
    def from_lists(cls, ad_emb, ad_key_off, ad_keys, field_card, cross_w, ad_begin: int = 0, device: int = 0,
                   stream=None):
        """Multi-valued ad fields: L given ad by ad as global key lists (ebr_build_index_lists)."""
        self = cls.__new__(cls)
        ad_emb = np.ascontiguousarray(ad_emb)
        self.dtype = BF16 if ad_emb.dtype == np.uint16 else F32
        if self.dtype == F32:
            ad_emb = np.ascontiguousarray(ad_emb, np.float32)
        off = np.ascontiguousarray(ad_key_off, np.int64)
        keys = np.ascontiguousarray(ad_keys, np.int32)
        field_card = np.ascontiguousarray(field_card, np.int32)
        cross_w = np.ascontiguousarray(cross_w, np.float32)
        n, self.d = ad_emb.shape
        self.n_fields = field_card.shape[0]
        self.n_keys = int(field_card.astype(np.int64).sum())
        self.ad_begin, self.n_ads, self.device = int(ad_begin), int(n), device
        h = ctypes.c_void_p()
        _check(_lib.ebr_build_index_lists(_np_ptr(ad_emb), self.dtype, self.ad_begin, self.ad_begin + n, self.d,
                                          _np_ptr(off), _np_ptr(keys), self.n_fields, _np_ptr(field_card),
                                          _np_ptr(cross_w), self.n_keys, device, _stream_ptr(stream),
                                          ctypes.byref(h)), "ebr_build_index_lists")
        self._h = h
        return self

    @classmethod
    def of(cls, inv, ad_begin: int = 0, device: int = 0, lo: int | None = None, hi: int | None = None,
           device_build: bool = False):
        lo = 0 if lo is None else lo
        hi = inv.n_ads if hi is None else hi
        return cls(inv.ad_emb[lo:hi], inv.ad_feat[lo:hi], inv.field_card, inv.cross_w,
                   ad_begin=ad_begin + lo, device=device, device_build=device_build)

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            _lib.ebr_free_index(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stats(self) -> dict:
        s = Stats()
        _check(_lib.ebr_index_stats(self._h, ctypes.byref(s)), "ebr_index_stats")
        return {k: getattr(s, k) for k, _ in Stats._fields_}

    def workspace_bytes(self, batch: int, slots: int, k: int) -> int:
        n = _lib.ebr_workspace_bytes(self._h, batch, slots, k)
        if n == 0:
            raise EbrError(1, "ebr_workspace_bytes")
        return int(n)

    def workspace_bytes_host(self, batch: int, slots: int, k: int) -> int:
        n = _lib.ebr_workspace_bytes_host(self._h, batch, slots, k)
        if n == 0:
            raise EbrError(1, "ebr_workspace_bytes_host")
        return int(n)

    def query_launches(self, batch: int, slots: int, k: int) -> int:
        return int(_lib.ebr_query_launches(self._h, batch, slots, k))

    def export(self, which: int) -> np.ndarray:
        """One device array of the index as uint32 (ebr_index_export; 0 key_chunk_off, 1
        key_word_off, 2 chunk_hdr, 3 chunk_last, 4 payload, 5 hot_mask)."""
        nb = ctypes.c_int64(0)
        _check(_lib.ebr_index_export(self.handle, which, None, 0, ctypes.byref(nb)), "ebr_index_export")
        out = np.zeros(nb.value // 4, np.uint32)
        if nb.value:
            _check(_lib.ebr_index_export(self.handle, which, _np_ptr(out), nb.value, ctypes.byref(nb)),
                   "ebr_index_export")
        return out

    def debug_decode(self, key: int) -> np.ndarray:
        n = _I64()
        st = _lib.ebr_debug_decode(self._h, key, None, 0, ctypes.byref(n))
        if st not in (0, 1):
            _check(st, "ebr_debug_decode")
        out = np.empty(max(int(n.value), 1), np.int32)
        _check(_lib.ebr_debug_decode(self._h, key, _np_ptr(out), out.shape[0], ctypes.byref(n)),
               "ebr_debug_decode")
        return out[: int(n.value)]


def score_topk(idx: Index, user_emb, user_feat, user_x, k: int, out_ids, out_scores, workspace,
               stream=None):
    """Device buffers (torch CUDA tensors); asynchronous on `stream`."""
    B, F, S = user_feat.shape
    _check(_lib.ebr_score_topk(idx.handle, _t_ptr(user_emb), B, _t_ptr(user_feat), _t_ptr(user_x),
                               S, k, _t_ptr(out_ids), _t_ptr(out_scores), _t_ptr(workspace),
                               workspace.numel() * workspace.element_size(), _stream_ptr(stream)),
           "ebr_score_topk")


def score_topk_keys(idx: Index, user_emb, user_feat, user_x, k: int, out_keys, workspace,
                    stream=None):
    B, F, S = user_feat.shape
    _check(_lib.ebr_score_topk_keys(idx.handle, _t_ptr(user_emb), B, _t_ptr(user_feat),
                                    _t_ptr(user_x), S, k, _t_ptr(out_keys), _t_ptr(workspace),
                                    workspace.numel() * workspace.element_size(),
                                    _stream_ptr(stream)),
           "ebr_score_topk_keys")


def score_topk_host(idx: Index, user_emb: np.ndarray, user_feat: np.ndarray, user_x: np.ndarray,
                    k: int, out_ids: np.ndarray, out_scores: np.ndarray, workspace, stream=None):
    """Host numpy buffers (ideally pinned); synchronous."""
    B, F, S = user_feat.shape
    _check(_lib.ebr_score_topk_host(idx.handle, _np_ptr(user_emb), B, _np_ptr(user_feat),
                                    _np_ptr(user_x), S, k, _np_ptr(out_ids), _np_ptr(out_scores),
                                    _t_ptr(workspace), workspace.numel() * workspace.element_size(),
                                    _stream_ptr(stream)),
           "ebr_score_topk_host")


def workspace_init(idx: Index, workspace, stream=None):
    _check(_lib.ebr_workspace_init(idx.handle, _t_ptr(workspace),
                                   workspace.numel() * workspace.element_size(), _stream_ptr(stream)),
           "ebr_workspace_init")


def new_workspace(idx: Index, batch: int, slots: int, k: int, host: bool = False, device=None):
    """Allocates (torch, uint8) and initialises a workspace for `idx`."""
    import torch
    n = idx.workspace_bytes_host(batch, slots, k) if host else idx.workspace_bytes(batch, slots, k)
    ws = torch.empty(n, dtype=torch.uint8, device=device if device is not None else f"cuda:{idx.device}")
    workspace_init(idx, ws)
    return ws


def query_error(workspace, stream=None) -> int:
    f = ctypes.c_uint32()
    st = _lib.ebr_query_error(_t_ptr(workspace), _stream_ptr(stream), ctypes.byref(f))
    if st not in (0, 5):
        _check(st, "ebr_query_error")
    return int(f.value)


def merge_topk(gathered, G: int, batch: int, k: int, out_ids, out_scores, stream=None):
    _check(_lib.ebr_merge_topk(_t_ptr(gathered), G, batch, k, _t_ptr(out_ids), _t_ptr(out_scores),
                               None, 0, _stream_ptr(stream)),
           "ebr_merge_topk")


def exchange_kth(local_keys, G: int, out_kq, stream=None):
    B, k = local_keys.shape
    _check(_lib.ebr_exchange_kth(_t_ptr(local_keys), B, k, G, _t_ptr(out_kq), _stream_ptr(stream)),
           "ebr_exchange_kth")


def exchange_pack(local_keys, kq_gathered, G: int, out_count, out_off, out_packed, stream=None):
    B, k = local_keys.shape
    _check(_lib.ebr_exchange_pack(_t_ptr(local_keys), B, k, _t_ptr(kq_gathered), G, _t_ptr(out_count),
                                  _t_ptr(out_off), _t_ptr(out_packed), _stream_ptr(stream)),
           "ebr_exchange_pack")


def merge_topk_packed(packed, counts, G: int, batch: int, k: int, out_ids, out_scores, stream=None):
    """packed: [G][stride] int64 (kappa bits), counts: [G][batch] int32 (uint32 bits)."""
    _check(_lib.ebr_merge_topk_packed(_t_ptr(packed), packed.shape[1], _t_ptr(counts), G, batch, k,
                                      _t_ptr(out_ids), _t_ptr(out_scores), _stream_ptr(stream)),
           "ebr_merge_topk_packed")


def encode_host(ad_feat: np.ndarray, field_card: np.ndarray):
    """Host-only encoder (no GPU): (key_chunk_off, key_word_off, chunk_hdr[2C], payload[W])."""
    ad_feat = np.ascontiguousarray(ad_feat, np.int32)
    field_card = np.ascontiguousarray(field_card, np.int32)
    n, F = ad_feat.shape
    M = int(field_card.astype(np.int64).sum())
    kco = np.empty(M + 1, np.uint32)
    kwo = np.empty(max(M, 1), np.uint32)
    C, W = _I64(), _I64()
    st = _lib.ebr_encode_host(_np_ptr(ad_feat), n, F, _np_ptr(field_card), M, _np_ptr(kco),
                              _np_ptr(kwo), None, 0, None, 0, ctypes.byref(C), ctypes.byref(W))
    if st != 0 and (st != 1 or C.value < 0):
        _check(st, "ebr_encode_host")
    hdr = np.zeros(2 * max(C.value, 1), np.uint32)
    pay = np.zeros(max(W.value, 1), np.uint32)
    _check(_lib.ebr_encode_host(_np_ptr(ad_feat), n, F, _np_ptr(field_card), M, _np_ptr(kco),
                                _np_ptr(kwo), _np_ptr(hdr), C.value, _np_ptr(pay), W.value,
                                ctypes.byref(C), ctypes.byref(W)),
           "ebr_encode_host")
    return kco, kwo[:M], hdr[: 2 * C.value], pay[: W.value]
