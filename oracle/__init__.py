"""CPU oracle for arXiv 2511.22460's Wide & Deep retrieval hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference) may
import this package.  The product path (paper_2511_22460_b200) never imports it and shares no
code with it; see ebr_oracle.c's header for what each function follows in the paper.

The C source is compiled on first use (gcc -O2 -fno-fast-math) into oracle/liboracle.so.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ebr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-std=c11", "-shared", "-fPIC",
                               "-pthread", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_scores_user.argtypes = [_I64, _I, _I, _P, _I, _P, _P, _P, _I64, _P, _I, _P, _P,
                                            _P, _P]
        _lib.oracle_wide_pairs_user.argtypes = [_I64, _I, _P, _P, _P, _I, _P, _P, _P]
        _lib.oracle_topk.argtypes = [_I64, _I, _I, _P, _I, _P, _P, _P, _I64, _I, _P, _I, _P, _P,
                                     _I, _I64, _I, _P, _P, _P]
        _lib.oracle_postings.argtypes = [_I64, _I, _P, _P, _I64, _P, _P]
        _lib.oracle_decode_chunks.argtypes = [_I64, _P, _P, _P, _P, _I64, _P, _P, _I64]
        _lib.oracle_ipnn_extend.argtypes = [_I64, _I, _I, _I, _I, _P, _P, _P, _P]
        _lib.oracle_scores_user_pairs.argtypes = [_I64, _I, _I, _P, _P, _P, _I, _P, _P, _I64, _P, _I, _P, _P,
                                                  _P, _P]
        for f in ("oracle_scores_user", "oracle_wide_pairs_user", "oracle_topk",
                  "oracle_postings", "oracle_decode_chunks", "oracle_ipnn_extend",
                  "oracle_scores_user_pairs"):
            getattr(_lib, f).restype = _I
    return _lib


def _c(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(_P)


def _emb(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint16:
        return a, 1
    return np.ascontiguousarray(a, np.float32), 0


class Oracle:
    """Holds one inventory (global ids id_base .. id_base+N-1) for repeated queries."""

    def __init__(self, ad_emb, ad_feat, field_card, cross_w, id_base: int = 0):
        self.ad_emb, self.is_bf16 = _emb(ad_emb)
        self.ad_feat, self._feat_p = _c(ad_feat, np.int32)
        self.field_card, self._card_p = _c(field_card, np.int32)
        self.cross_w, self._w_p = _c(cross_w, np.float32)
        self.n_ads, self.d = self.ad_emb.shape
        self.n_fields = self.field_card.shape[0]
        self.n_keys = int(self.field_card.astype(np.int64).sum())
        self.id_base = int(id_base)

    @classmethod
    def of(cls, inv, id_base: int = 0):
        return cls(inv.ad_emb, inv.ad_feat, inv.field_card, inv.cross_w, id_base)

    def scores(self, user_emb, user_feat, user_x):
        """Scorer A for one user: (r[N] fp64, sigma[N] fp64)."""
        ue, ub = _emb(np.asarray(user_emb).reshape(1, -1))
        assert ub == self.is_bf16
        uf, ufp = _c(user_feat, np.int32)
        ux, uxp = _c(user_x, np.float32)
        slots = uf.shape[-1]
        r = np.empty(self.n_ads, np.float64)
        s = np.empty(self.n_ads, np.float64)
        rc = lib().oracle_scores_user(self.n_ads, self.d, self.is_bf16, self.ad_emb.ctypes.data,
                                      self.n_fields, self._feat_p, self._card_p, self._w_p,
                                      self.n_keys, ue.ctypes.data, slots, ufp, uxp,
                                      r.ctypes.data, s.ctypes.data)
        if rc:
            raise ValueError(f"oracle_scores_user rc={rc}")
        return r, s

    def wide_pairs(self, user_feat, user_x):
        """Scorer B (explicit feature-pair enumeration), wide term only, one user."""
        uf, ufp = _c(user_feat, np.int32)
        ux, uxp = _c(user_x, np.float32)
        out = np.empty(self.n_ads, np.float64)
        rc = lib().oracle_wide_pairs_user(self.n_ads, self.n_fields, self._feat_p, self._card_p,
                                          self._w_p, uf.shape[-1], ufp, uxp, out.ctypes.data)
        if rc:
            raise ValueError(f"oracle_wide_pairs_user rc={rc}")
        return out

    def topk(self, user_emb, user_feat, user_x, k: int, threads: int = 1):
        """(ids[B][K] int32, r[B][K] fp64, sigma[B][K] fp64), sorted by (r desc, id asc)."""
        ue, ub = _emb(user_emb)
        assert ub == self.is_bf16
        uf, ufp = _c(user_feat, np.int32)
        ux, uxp = _c(user_x, np.float32)
        B, slots = uf.shape[0], uf.shape[-1]
        ids = np.empty((B, k), np.int32)
        r = np.empty((B, k), np.float64)
        s = np.empty((B, k), np.float64)
        rc = lib().oracle_topk(self.n_ads, self.d, self.is_bf16, self.ad_emb.ctypes.data,
                               self.n_fields, self._feat_p, self._card_p, self._w_p, self.n_keys,
                               B, ue.ctypes.data, slots, ufp, uxp, k, self.id_base, threads,
                               ids.ctypes.data, r.ctypes.data, s.ctypes.data)
        if rc:
            raise ValueError(f"oracle_topk rc={rc}")
        return ids, r, s

    def postings(self):
        """Inverted list of L: (offsets[M+1] int64, ads[nnz] int32), local ad ids ascending."""
        off = np.empty(self.n_keys + 1, np.int64)
        rc = lib().oracle_postings(self.n_ads, self.n_fields, self._feat_p, self._card_p,
                                   self.n_keys, off.ctypes.data, None)
        if rc:
            raise ValueError(f"oracle_postings rc={rc}")
        ads = np.empty(int(off[-1]), np.int32)
        rc = lib().oracle_postings(self.n_ads, self.n_fields, self._feat_p, self._card_p,
                                   self.n_keys, off.ctypes.data, ads.ctypes.data)
        if rc:
            raise ValueError(f"oracle_postings rc={rc}")
        return off, ads


def decode_chunks(key_chunk_off, key_word_off, chunk_hdr, payload, cap: int):
    """Independent decoder of the documented posting-chunk wire format -> (offsets, ads)."""
    kco, kcop = _c(key_chunk_off, np.uint32)
    kwo, kwop = _c(key_word_off, np.uint32)
    hdr, hdrp = _c(chunk_hdr, np.uint32)
    pay, payp = _c(payload, np.uint32)
    n_keys = kco.shape[0] - 1
    off = np.empty(n_keys + 1, np.int64)
    ads = np.empty(max(cap, 1), np.int32)
    rc = lib().oracle_decode_chunks(n_keys, kcop, kwop, hdrp, payp, pay.shape[0], off.ctypes.data,
                                    ads.ctypes.data, cap)
    if rc:
        raise ValueError(f"oracle_decode_chunks rc={rc}")
    return off, ads[: int(off[-1])]


def ipnn_extend(h, u, W):
    """IPNN extension (Eq. 7-8): [h, W u] per row in fp64.  h: [rows][d0] fp32 or bf16
    bits (uint16); u: [rows][n] fp32; W: [d1][n] fp32."""
    h = np.ascontiguousarray(h)
    is_bf16 = 1 if h.dtype == np.uint16 else 0
    if not is_bf16:
        h = np.ascontiguousarray(h, np.float32)
    u = np.ascontiguousarray(u, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    rows, d0 = h.shape
    d1, n = W.shape
    out = np.empty((rows, d0 + d1), np.float64)
    rc = lib().oracle_ipnn_extend(rows, d0, n, d1, is_bf16, h.ctypes.data, u.ctypes.data, W.ctypes.data,
                                  out.ctypes.data)
    if rc:
        raise ValueError(f"oracle_ipnn_extend rc={rc}")
    return out


class OraclePairs:
    """Scorer A for an inventory whose L is given ad by ad as key lists (multi-valued fields):
    ad_key_off [N+1] int64, ad_keys [nnz] int32 (global keys base_f + v)."""

    def __init__(self, ad_emb, ad_key_off, ad_keys, field_card, cross_w):
        self.ad_emb, self.is_bf16 = _emb(ad_emb)
        self.off = np.ascontiguousarray(ad_key_off, np.int64)
        self.keys = np.ascontiguousarray(ad_keys, np.int32)
        self.field_card = np.ascontiguousarray(field_card, np.int32)
        self.cross_w = np.ascontiguousarray(cross_w, np.float32)
        self.n_ads, self.d = self.ad_emb.shape
        self.n_keys = int(self.field_card.astype(np.int64).sum())

    def scores(self, user_emb, user_feat, user_x):
        ue, ub = _emb(np.asarray(user_emb).reshape(1, -1))
        assert ub == self.is_bf16
        uf = np.ascontiguousarray(user_feat, np.int32)
        ux = np.ascontiguousarray(user_x, np.float32)
        r = np.empty(self.n_ads, np.float64)
        s = np.empty(self.n_ads, np.float64)
        rc = lib().oracle_scores_user_pairs(self.n_ads, self.d, self.is_bf16, self.ad_emb.ctypes.data,
                                            self.off.ctypes.data, self.keys.ctypes.data,
                                            self.field_card.shape[0], self.field_card.ctypes.data,
                                            self.cross_w.ctypes.data, self.n_keys, ue.ctypes.data,
                                            uf.shape[-1], uf.ctypes.data, ux.ctypes.data, r.ctypes.data,
                                            s.ctypes.data)
        if rc:
            raise ValueError(f"oracle_scores_user_pairs rc={rc}")
        return r, s
