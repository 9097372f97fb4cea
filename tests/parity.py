"""Comparison rules between the CUDA path's top-K and the CPU oracle (test infrastructure).

exact mode  (dyadic inputs: every partial sum is exact in fp32): ids and scores
            must be bit-identical to the oracle's (score desc, id asc) order.
real mode   scores within tol * sigma(a) of the oracle's fp64 value (sigma = sum of |terms|,
            DESIGN.md reading R12), and the tie-aware set rule:
              - every oracle id with r > s_K + tau(a) + tau_K must be returned,
              - every returned id must have r >= s_K - tau(a) - tau_K,
              - consecutive outputs ordered within tau.
"""
from __future__ import annotations

import numpy as np

TOL_F32 = 1e-5      # north star: 1e-5 relative in fp32 (also bf16 inputs vs the same bf16 values)


def oracle_full(o, users, b):
    return o.scores(users.user_emb[b], users.user_feat[b], users.user_x[b])


def topk_order(r, kk):
    """The first kk ads of the (score desc, id asc) order of r."""
    n = r.shape[0]
    if n > 4 * kk + 1024:
        # O(n): every ad at or above the kk-th largest score (ties included), then the exact
        # order of that subset -- the same prefix as the full lexsort
        s_k = np.partition(r, n - kk)[n - kk]
        sub = np.nonzero(r >= s_k)[0]
        return sub[np.lexsort((sub, -r[sub]))][:kk]
    return np.lexsort((np.arange(n), -r))[:kk]


def check_many(o, users, ids, sc, k, mode, sel=None, threads=None, id_base=0):
    """check_user for the users `sel` (default all), oracle scoring in a thread pool (the ctypes
    oracle call and numpy's partition release the GIL).  Returns the summed id mismatches."""
    import concurrent.futures as cf
    import os
    sel = list(range(users.batch)) if sel is None else list(sel)
    threads = threads or min(len(sel), os.cpu_count() or 1)

    def one(b):
        r, s = o.scores(users.user_emb[b], users.user_feat[b], users.user_x[b])
        return check_user(ids[b], sc[b], r, s, k, mode, id_base=id_base)
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        return sum(ex.map(one, sel))


def check_user(ids, scores, r, sigma, k, mode, tol=TOL_F32, id_base=0):
    """ids/scores: one user's GPU output (k,); r/sigma: oracle fp64 arrays over the inventory."""
    n = r.shape[0]
    kk = min(k, n)
    order = topk_order(r, kk)
    ids = np.asarray(ids)
    scores = np.asarray(scores)
    # padding
    assert (ids[kk:] == -1).all(), "padding ids"
    assert np.isneginf(scores[kk:]).all(), "padding scores"
    ids, scores = ids[:kk], scores[:kk]
    loc = ids - id_base
    assert ((loc >= 0) & (loc < n)).all(), "id out of range"
    assert len(np.unique(loc)) == kk, "duplicate ids"
    if mode == "exact":
        assert (loc == order).all(), f"ids differ at {np.nonzero(loc != order)[0][:10]}"
        assert (scores.astype(np.float64) == r[order]).all(), "scores differ"
        return 0
    tau = tol * sigma + 1e-30
    err = np.abs(scores.astype(np.float64) - r[loc])
    assert (err <= tau[loc]).all(), f"score error {(err / tau[loc]).max():.3g} x tol"
    sK = r[order[kk - 1]]
    tK = tau[order[kk - 1]]
    must = order[r[order] > sK + tau[order] + tK]
    assert np.isin(must, loc).all(), "a clear top-K ad is missing"
    assert (r[loc] >= sK - tau[loc] - tK).all(), "a returned ad is clearly below the K-th"
    assert (np.diff(scores) <= 0).all(), "output not sorted by its own scores"
    rr = r[loc]
    assert (rr[1:] <= rr[:-1] + tau[loc][1:] + tau[loc][:-1]).all(), "order violated beyond tolerance"
    return int((loc != order).sum())
