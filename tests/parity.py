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


def check_user(ids, scores, r, sigma, k, mode, tol=TOL_F32, id_base=0):
    """ids/scores: one user's GPU output (k,); r/sigma: oracle fp64 arrays over the inventory."""
    n = r.shape[0]
    order = np.lexsort((np.arange(n), -r))[:k]
    kk = min(k, n)
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
