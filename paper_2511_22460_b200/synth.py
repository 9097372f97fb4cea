"""Seeded synthetic workload generator (inputs only; holds none of the method's arithmetic).

Shared by the CUDA path's tests/bench and by the oracle's tests: it produces the raw inputs of
the C-ABI (ad embeddings, ad feature values, field cardinalities, the cross-weight table, user
embeddings, user feature values and statistics).  It never computes a key, a weight product, a
score or a ranking -- those belong to each side separately.

Recipe, shaped by the paper's wide features:
  * side information with hierarchical categories of low cardinality up to item ids of ~N
    cardinality (§3.3, l.248: "multi-level ad categories, tags, advertiser IDs, and item
    IDs"), so field cardinalities are log-spaced  V_f = min(N, round(2^(4 + 16 f/(F-1)))).
  * ad values Zipf(alpha)-popular through a fixed per-field permutation (hot values are not low
    ids); an ad's field is empty with probability 0.1 (L_{a,i}=0, Eq. 9, l.252).
  * user values are "statistically aggregated" behaviour over ads the user interacted with
    (§4.1.2, l.387), so each user x field draws S distinct values by the same
    popularity (hot features are queried often), each slot emptied with probability 0.25.
  * modes: "exact" (dyadic values: every partial sum is exact in fp32) and
    "real" (h ~ N(0,1) d^-1/4, w ~ N(0, 0.5^2), x ~ U(0,1]).
  * bf16 embeddings are produced here already rounded (round-to-nearest-even) and handed to both
    sides as raw bf16 bit patterns: the library never converts fp32 -> bf16.
"""
from __future__ import annotations

import dataclasses
import os

import numpy as np

SEED_BASE = 2511_22460


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n_ads: int
    d: int
    dtype: str          # "f32" | "bf16"
    n_fields: int
    alpha: float
    batch: int
    k: int
    slots: int = 2
    cfg_id: int = 0     # seed namespace


# BASELINE.json configs.  C5 is a sweep; its preset is one point.
CONFIGS = {
    "C1": Config("C1", 10_000, 64, "f32", 8, 1.0, 1, 100, cfg_id=1),
    "C2": Config("C2", 1_000_000, 64, "f32", 32, 1.0, 1, 500, cfg_id=2),
    "C3": Config("C3", 10_000_000, 128, "bf16", 32, 1.0, 256, 1000, cfg_id=3),
    "C4": Config("C4", 5_000_000, 64, "bf16", 64, 1.2, 64, 1000, cfg_id=4),
    "C5": Config("C5", 20_000_000, 128, "bf16", 32, 1.0, 256, 1000, cfg_id=5),
}


@dataclasses.dataclass
class Inventory:
    n_ads: int
    d: int
    dtype: str
    ad_emb: np.ndarray       # [N][d] float32, or uint16 (bf16 bit patterns)
    ad_feat: np.ndarray      # [N][F] int32, -1 = empty
    field_card: np.ndarray   # [F] int32
    cross_w: np.ndarray      # [M] float32, M = sum(field_card)
    perm_seed: int = 0       # seed of the per-field popularity permutations (shared with users)


@dataclasses.dataclass
class Users:
    batch: int
    slots: int
    user_emb: np.ndarray     # [B][d] same dtype as the inventory
    user_feat: np.ndarray    # [B][F][S] int32, -1 = empty slot
    user_x: np.ndarray       # [B][F][S] float32 (0 where empty)


def field_cards(n_ads: int, n_fields: int) -> np.ndarray:
    """V_f = min(N, round(2^(4+16 f/(F-1)))), log-spaced 16 .. 2^20."""
    if n_fields == 1:
        e = np.array([4.0])
    else:
        e = 4.0 + 16.0 * np.arange(n_fields) / (n_fields - 1)
    v = np.minimum(n_ads, np.round(2.0 ** e)).astype(np.int64)
    return np.maximum(v, 1).astype(np.int32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    out = np.empty(u.shape, dtype=np.uint16)
    fo, fu = out.reshape(-1), u.reshape(-1)
    step = 1 << 24
    for lo in range(0, fu.size, step):       # uint32 is enough: finite inputs stay below 2^32
        c = fu[lo:lo + step]
        r = (c >> 16) & np.uint32(1)
        r += c
        r += np.uint32(0x7FFF)
        r >>= 16
        fo[lo:lo + step] = r
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


class _Zipf:
    """Inverse-CDF sampler for P(r) ∝ (r+1)^-alpha on [0, V), composed with a permutation."""

    def __init__(self, v: int, alpha: float, perm: np.ndarray):
        p = (np.arange(1, v + 1, dtype=np.float64)) ** (-alpha)
        c = np.cumsum(p)
        self.cdf = c / c[-1]
        self.cdf[-1] = 1.0
        self.perm = perm
        self.v = v

    def draw(self, u: np.ndarray) -> np.ndarray:
        r = np.searchsorted(self.cdf, u, side="right")
        np.minimum(r, self.v - 1, out=r)
        return self.perm[r]


def _embeddings(rng: np.random.Generator, n: int, d: int, mode: str) -> np.ndarray:
    if mode == "exact":
        return (rng.integers(-8, 9, size=(n, d), dtype=np.int8).astype(np.float32) / 16.0)
    return (rng.standard_normal((n, d), dtype=np.float32) * np.float32(d ** -0.25))


def _samplers(cards: np.ndarray, alpha: float, seed: int) -> list:
    prng = np.random.default_rng(seed + 7)
    return [_Zipf(int(v), alpha, prng.permutation(int(v)).astype(np.int32)) for v in cards]


def make_inventory(n_ads: int, d: int, n_fields: int, alpha: float = 1.0, dtype: str = "f32",
                   mode: str = "real", seed: int = 0, p_empty: float = 0.1,
                   cards: np.ndarray | None = None) -> Inventory:
    rng = np.random.default_rng(seed)
    cards = field_cards(n_ads, n_fields) if cards is None else np.asarray(cards, np.int32)
    samp = _samplers(cards, alpha, seed)
    M = int(cards.sum())
    if mode == "exact":
        w = rng.integers(-32, 33, size=M).astype(np.float32) / 32.0
    else:
        w = (rng.standard_normal(M, dtype=np.float32) * np.float32(0.5))
    feat = np.empty((n_ads, n_fields), dtype=np.int32)
    step = 1 << 20
    for lo in range(0, n_ads, step):
        hi = min(n_ads, lo + step)
        for f in range(n_fields):
            u = rng.random(hi - lo)
            col = samp[f].draw(u).astype(np.int32)
            col[rng.random(hi - lo) < p_empty] = -1
            feat[lo:hi, f] = col
    emb = np.empty((n_ads, d), dtype=np.float32)
    for lo in range(0, n_ads, step):
        hi = min(n_ads, lo + step)
        emb[lo:hi] = _embeddings(rng, hi - lo, d, mode)
    if dtype == "bf16":
        emb = f32_to_bf16_bits(emb)
    return Inventory(n_ads, d, dtype, emb, feat, cards, w, seed)


def make_users(inv: Inventory, batch: int, slots: int = 2, alpha: float = 1.0, mode: str = "real",
               seed: int = 1, p_empty: float = 0.25) -> Users:
    rng = np.random.default_rng(seed)
    F = inv.field_card.shape[0]
    samp = _samplers(inv.field_card, alpha, inv.perm_seed)
    feat = np.empty((batch, F, slots), dtype=np.int32)
    for f in range(F):
        v = samp[f].draw(rng.random((batch, slots)))
        # distinct within (u, f): redraw duplicates (bounded; cardinality >= 16 > slots)
        for _ in range(64):
            dup = np.zeros_like(v, dtype=bool)
            for s in range(1, slots):
                dup[:, s] = (v[:, :s] == v[:, s:s + 1]).any(axis=1)
            if not dup.any():
                break
            v[dup] = samp[f].draw(rng.random(int(dup.sum())))
        else:  # pragma: no cover - only for degenerate tiny cardinalities
            for s in range(1, slots):
                bad = (v[:, :s] == v[:, s:s + 1]).any(axis=1)
                v[bad, s] = -1
        feat[:, f, :] = v
    feat[rng.random(feat.shape) < p_empty] = -1
    if mode == "exact":
        x = rng.integers(1, 17, size=feat.shape).astype(np.float32) / 16.0
    else:
        x = (1.0 - rng.random(feat.shape)).astype(np.float32)   # U(0,1]
    x[feat < 0] = 0.0
    emb = _embeddings(rng, batch, inv.d, mode)
    if inv.dtype == "bf16":
        emb = f32_to_bf16_bits(emb)
    return Users(batch, slots, emb, feat, x)


def make_config(cfg: Config | str, mode: str = "real", n_ads: int | None = None,
                batch: int | None = None, seed_offset: int = 0):
    """Inventory + users for a named config (optionally shrunk for parity tests)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    n = cfg.n_ads if n_ads is None else n_ads
    b = cfg.batch if batch is None else batch
    base = SEED_BASE + 100 * cfg.cfg_id + 10_000 * seed_offset
    cache = os.environ.get("EBR_SYNTH_CACHE")     # optional directory: reuse a generated inventory
    path = os.path.join(cache, f"{cfg.name}_{n}_{mode}_{base}.npz") if cache else None
    if path and os.path.exists(path):
        z = np.load(path)
        inv = Inventory(n, cfg.d, cfg.dtype, z["emb"], z["feat"], z["cards"], z["w"], int(z["seed"]))
    else:
        inv = make_inventory(n, cfg.d, cfg.n_fields, cfg.alpha, cfg.dtype, mode, seed=base + 0)
        if path:
            os.makedirs(cache, exist_ok=True)
            tmp = f"{path}.{os.getpid()}.tmp.npz"          # (concurrent writers: one file each)
            np.savez(tmp, emb=inv.ad_emb, feat=inv.ad_feat, cards=inv.field_card, w=inv.cross_w,
                     seed=inv.perm_seed)
            os.replace(tmp, path)
    users = make_users(inv, b, cfg.slots, cfg.alpha, mode, seed=base + 1)
    return inv, users
