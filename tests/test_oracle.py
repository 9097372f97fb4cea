"""Pins for the CPU oracle (-m "not gpu").  Each test checks the oracle against something other
than itself: values the spec/paper fix (golden fixtures with citations), hand-worked values,
closed forms, textbook routines (numpy matmul / lexsort / nonzero), and invariants (linearity,
conservation, scorer A == scorer B, permutation invariance).  No expected value here comes from
the CUDA path."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2511_22460_b200 import synth


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def _zero_emb(n, d=1):
    return np.zeros((n, d), np.float32)


# ---------------------------------------------------------------- golden: SPEC worked example

def test_spec_worked_example_wide(golden_dir):
    g = _load(golden_dir, "spec_oracle_example.json")
    ad_feat = np.array(g["ad_feat"], np.int32)
    o = oracle.Oracle(_zero_emb(3), ad_feat, g["field_card"], g["cross_w"])
    uf = np.array(g["user_feat"], np.int32)
    ux = np.array(g["user_x"], np.float32)
    r, _ = o.scores(np.zeros(1, np.float32), uf, ux)
    assert r.tolist() == g["expected_wide"]            # exact in fp32 and fp64
    assert o.wide_pairs(uf, ux).tolist() == g["expected_wide"]
    ids, sc, _ = o.topk(np.zeros((1, 1), np.float32), uf[None], ux[None], 2)
    assert ids[0].tolist() == g["expected_topk_k2"]["ids"]
    assert sc[0].tolist() == g["expected_topk_k2"]["scores"]


def test_spec_empty_query_and_identity_L():
    # S:110 empty query -> all zeros; S:111 identity-like L -> a single spike.
    n = 5
    feat = np.full((n, n), -1, np.int32)
    np.fill_diagonal(feat, 0)                          # ad i has only key i
    o = oracle.Oracle(_zero_emb(n), feat, [1] * n, np.arange(1, n + 1, dtype=np.float32))
    empty = np.full((n, 1), -1, np.int32)
    r, _ = o.scores(np.zeros(1, np.float32), empty, np.zeros((n, 1), np.float32))
    assert (r == 0).all()
    q = empty.copy()
    q[3, 0] = 0
    x = np.zeros((n, 1), np.float32)
    x[3, 0] = 0.5
    r, _ = o.scores(np.zeros(1, np.float32), q, x)
    assert r.tolist() == [0, 0, 0, 4 * 0.5, 0]


def test_spec_fused_example():
    # S:356 fused = tower part + hitmatch part: 0.3 + 3.5 = 3.8 for ad2 of the S:109 example.
    feat = np.array([[0, -1, 0, -1], [-1, 0, -1, -1], [0, 0, -1, 0]], np.int32)
    emb = np.array([[0.0], [0.0], [0.3]], np.float32)
    o = oracle.Oracle(emb, feat, [1, 1, 1, 1], [0.5, 2.0, 7.0, 1.0])
    r, _ = o.scores(np.ones(1, np.float32), np.array([[0], [0], [-1], [0]], np.int32),
                    np.array([[1], [1], [0], [1]], np.float32))
    assert abs(r[2] - 3.8) < 1e-7
    assert r[2] == float(np.float32(0.3)) + 3.5


# ---------------------------------------------------------------- golden: hand-worked inventory

def test_hand_inventory(golden_dir):
    g = _load(golden_dir, "hand_inventory.json")
    o = oracle.Oracle(np.array(g["ad_emb"], np.float32), np.array(g["ad_feat"], np.int32),
                      g["field_card"], g["cross_w"])
    uf = np.array(g["user_feat"], np.int32)
    ux = np.array(g["user_x"], np.float32)
    r, s = o.scores(np.array(g["user_emb"], np.float32), uf, ux)
    assert r.tolist() == g["expected_scores"]
    assert s.tolist() == g["expected_sigma"]
    ue = np.array([g["user_emb"]], np.float32)
    ids, sc, _ = o.topk(ue, uf[None], ux[None], 2)
    assert ids[0].tolist() == g["expected_top2_ids"]
    ids, sc, _ = o.topk(ue, uf[None], ux[None], 4)
    assert ids[0].tolist() == g["expected_top4_ids"]
    ids, sc, _ = o.topk(ue, uf[None], ux[None], 6)     # K > N pads with (-1, -inf) (R15)
    assert ids[0].tolist() == g["expected_top4_ids"] + [-1, -1]
    assert np.isneginf(sc[0, 4:]).all()


# ---------------------------------------------------------------- top-K rules

def test_topk_ties_ascending_id_and_full_sort():
    # S:367 all-equal scores, k=2 -> ads 0 and 1; k=N -> full sort.
    n = 6
    feat = np.zeros((n, 1), np.int32)
    o = oracle.Oracle(_zero_emb(n), feat, [1], [1.0])
    uf = np.zeros((1, 1, 1), np.int32)
    ux = np.ones((1, 1, 1), np.float32)
    ids, sc, _ = o.topk(np.zeros((1, 1), np.float32), uf, ux, 2)
    assert ids[0].tolist() == [0, 1] and sc[0].tolist() == [1.0, 1.0]


def test_topk_full_sort_equals_lexsort():
    inv, us = synth.make_config("C1", mode="exact", n_ads=3000, batch=2)
    o = oracle.Oracle.of(inv)
    ids, sc, _ = o.topk(us.user_emb, us.user_feat, us.user_x, inv.n_ads)
    for b in range(2):
        r, _ = o.scores(us.user_emb[b], us.user_feat[b], us.user_x[b])
        order = np.lexsort((np.arange(inv.n_ads), -r))    # textbook: score desc, id asc
        assert (ids[b] == order).all()
        assert (sc[b] == r[order]).all()
        assert len(np.unique(r)) < inv.n_ads             # exact mode really has ties


def test_topk_permutation_invariance():
    # selection is invariant to input order (real mode: no ties).
    inv, us = synth.make_config("C1", mode="real", n_ads=2000, batch=1)
    o = oracle.Oracle.of(inv)
    ids, sc, _ = o.topk(us.user_emb, us.user_feat, us.user_x, 50)
    perm = np.random.default_rng(5).permutation(inv.n_ads)
    o2 = oracle.Oracle(inv.ad_emb[perm], inv.ad_feat[perm], inv.field_card, inv.cross_w)
    ids2, sc2, _ = o2.topk(us.user_emb, us.user_feat, us.user_x, 50)
    assert (perm[ids2[0]] == ids[0]).all()
    assert (sc2 == sc).all()


def test_topk_id_base_and_threads():
    inv, us = synth.make_config("C1", mode="exact", n_ads=1500, batch=5)
    o = oracle.Oracle.of(inv)
    ids1, sc1, _ = o.topk(us.user_emb, us.user_feat, us.user_x, 37, threads=1)
    ids4, sc4, _ = o.topk(us.user_emb, us.user_feat, us.user_x, 37, threads=4)
    assert (ids1 == ids4).all() and (sc1 == sc4).all()
    ob = oracle.Oracle(inv.ad_emb, inv.ad_feat, inv.field_card, inv.cross_w, id_base=1000)
    idsb, scb, _ = ob.topk(us.user_emb, us.user_feat, us.user_x, 37)
    assert (idsb == ids1 + 1000).all() and (scb == sc1).all()


# ---------------------------------------------------------------- deep term vs textbook GEMM

@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_deep_term_equals_numpy_matmul(dtype):
    inv = synth.make_inventory(700, 48, 3, dtype=dtype, mode="real", seed=11)
    us = synth.make_users(inv, 3, seed=12)
    o = oracle.Oracle.of(inv)
    A = inv.ad_emb if dtype == "f32" else synth.bf16_bits_to_f32(inv.ad_emb)
    U = us.user_emb if dtype == "f32" else synth.bf16_bits_to_f32(us.user_emb)
    empty = np.full(us.user_feat.shape[1:], -1, np.int32)
    for b in range(3):
        r, s = o.scores(us.user_emb[b], empty, np.zeros(empty.shape, np.float32))
        ref = A.astype(np.float64) @ U[b].astype(np.float64)
        assert np.allclose(r, ref, rtol=0, atol=1e-12)
        assert np.allclose(s, np.abs(A.astype(np.float64) * U[b].astype(np.float64)).sum(1),
                           rtol=1e-14, atol=0)


def test_bf16_widening_known_patterns():
    emb = np.array([[0x3F80], [0xC000], [0x3E80], [0x8000]], np.uint16)   # 1, -2, 0.25, -0
    o = oracle.Oracle(emb, np.full((4, 1), -1, np.int32), [1], [0.0])
    r, _ = o.scores(np.array([0x3F80], np.uint16), np.full((1, 1), -1, np.int32),
                    np.zeros((1, 1), np.float32))
    assert r.tolist() == [1.0, -2.0, 0.25, 0.0]


# ---------------------------------------------------------------- wide term: A == B, invariants

@pytest.mark.parametrize("mode", ["exact", "real"])
def test_scorer_a_equals_pair_enumeration(mode):
    inv, us = synth.make_config("C1", mode=mode, n_ads=4000, batch=3)
    o = oracle.Oracle(np.zeros((inv.n_ads, 1), np.float32), inv.ad_feat, inv.field_card,
                      inv.cross_w)
    for b in range(3):
        r, _ = o.scores(np.zeros(1, np.float32), us.user_feat[b], us.user_x[b])
        w = o.wide_pairs(us.user_feat[b], us.user_x[b])
        if mode == "exact":
            assert (r == w).all()
        else:
            assert np.allclose(r, w, rtol=1e-12, atol=1e-300)
        assert np.count_nonzero(w) > 0


def test_wide_linearity_and_conservation():
    # S:115 linearity; S:277 conservation: sum_a wide(a) = sum_k w~_k |posting_k|.
    inv, us = synth.make_config("C1", mode="exact", n_ads=5000, batch=1)
    o = oracle.Oracle(np.zeros((inv.n_ads, 1), np.float32), inv.ad_feat, inv.field_card,
                      inv.cross_w)
    uf, ux = us.user_feat[0], us.user_x[0]
    r, _ = o.scores(np.zeros(1, np.float32), uf, ux)
    r2, _ = o.scores(np.zeros(1, np.float32), uf, 2 * ux)
    assert (r2 == 2 * r).all()
    base = np.concatenate([[0], np.cumsum(inv.field_card)[:-1]])
    total = 0.0
    for f in range(uf.shape[0]):
        for s in range(uf.shape[1]):
            v = uf[f, s]
            if v < 0:
                continue
            count = int((inv.ad_feat[:, f] == v).sum())        # |posting_k| by numpy
            total += float(inv.cross_w[base[f] + v]) * float(ux[f, s]) * count
    assert r.sum() == total


def test_duplicate_slot_is_additive():
    # Reading R3: the same (f, v) twice in one user adds.
    feat = np.array([[0], [1]], np.int32)
    o = oracle.Oracle(_zero_emb(2), feat, [2], [1.0, 10.0])
    uf = np.array([[0, 0]], np.int32)
    ux = np.array([[0.5, 0.25]], np.float32)
    r, _ = o.scores(np.zeros(1, np.float32), uf, ux)
    assert r.tolist() == [0.75, 0.0]
    assert o.wide_pairs(uf, ux).tolist() == [0.75, 0.0]


def test_bad_values_rejected():
    o = oracle.Oracle(_zero_emb(2), np.array([[0], [1]], np.int32), [2], [1.0, 1.0])
    with pytest.raises(ValueError):
        o.scores(np.zeros(1, np.float32), np.array([[2]], np.int32), np.ones((1, 1), np.float32))
    with pytest.raises(ValueError):
        oracle.Oracle(_zero_emb(1), np.array([[5]], np.int32), [2], [1.0, 1.0]).postings()


# ---------------------------------------------------------------- posting lists and decoder

def test_postings_equal_numpy_nonzero():
    inv = synth.make_inventory(3000, 4, 6, alpha=1.2, seed=3)
    o = oracle.Oracle.of(inv)
    off, ads = o.postings()
    base = np.concatenate([[0], np.cumsum(inv.field_card)[:-1]])
    for f in range(6):
        for v in range(inv.field_card[f]):
            k = base[f] + v
            ref = np.nonzero(inv.ad_feat[:, f] == v)[0]
            assert (ads[off[k]:off[k + 1]] == ref).all()
    assert off[-1] == (inv.ad_feat >= 0).sum()


def test_decoder_hand_trace(golden_dir):
    g = _load(golden_dir, "wire_format_example.json")
    assert [int(h, 16) for h in g["payload_hex"]] == g["payload"]
    off, ads = oracle.decode_chunks(g["key_chunk_off"], g["key_word_off"], g["chunk_hdr"],
                                    g["payload"], cap=64)
    assert off.tolist() == [0, 7] and ads.tolist() == g["list"]


def test_decoder_special_chunks():
    # n=1 chunk (no payload), b=0 consecutive run (no payload words), two keys, relative offsets.
    kco = [0, 1, 3]
    kwo = [0, 0]
    hdr = [7, 0,                      # key0: single posting 7
           10, (31) | (0 << 5),       # key1 chunk0: 32 consecutive ids 10..41, b = 0
           50, 2 | (4 << 5) | (0 << 10)]   # key1 chunk1: 50, +3, +16 (gap-1 = 2, 15; b=4)
    payload = [2 | (15 << 4), 0]
    off, ads = oracle.decode_chunks(kco, kwo, hdr, payload, cap=64)
    assert off.tolist() == [0, 1, 36]
    assert ads.tolist() == [7] + list(range(10, 42)) + [50, 53, 69]


# ---- NEXT-4: the IPNN extension h~ = [h, W u] (Eq. 7-8)

def test_ipnn_extend_hand_example_and_numpy():
    W = np.array([[1, 2], [3, 4]], np.float32)
    u = np.array([[1, 1], [0.5, -2]], np.float32)
    h = np.array([[0.5], [-1.0]], np.float32)
    out = oracle.ipnn_extend(h, u, W)
    assert (out == np.array([[0.5, 3, 7], [-1.0, -3.5, -6.5]])).all()      # worked by hand
    rng = np.random.default_rng(7)
    h = rng.standard_normal((5, 9)).astype(np.float32)
    u = rng.standard_normal((5, 33)).astype(np.float32)
    W = rng.standard_normal((12, 33)).astype(np.float32)
    out = oracle.ipnn_extend(h, u, W)
    assert (out[:, :9] == h.astype(np.float64)).all()
    assert np.allclose(out[:, 9:], u.astype(np.float64) @ W.astype(np.float64).T, rtol=1e-13, atol=1e-12)
    # bf16 tower outputs are widened exactly
    hb = np.array([[0x3F80, 0xC000]], np.uint16)                     # 1.0, -2.0
    assert (oracle.ipnn_extend(hb, np.zeros((1, 1), np.float32), np.zeros((1, 1), np.float32))[0, :2]
            == [1.0, -2.0]).all()


# ---- NEXT-4: multi-valued ad fields (L given ad by ad as key lists)

def test_pairs_scorer_equals_single_valued_and_hand_example():
    inv, users = synth.make_config("C1", mode="exact", n_ads=500, batch=2)
    base = np.concatenate([[0], np.cumsum(inv.field_card)[:-1]]).astype(np.int64)
    keys = [[int(base[f] + v) for f, v in enumerate(row) if v >= 0] for row in inv.ad_feat]
    off = np.concatenate([[0], np.cumsum([len(k) for k in keys])]).astype(np.int64)
    flat = np.array([k for ks in keys for k in ks], np.int32)
    a, p = oracle.Oracle.of(inv), oracle.OraclePairs(inv.ad_emb, off, flat, inv.field_card, inv.cross_w)
    for b in range(2):
        ra, sa = a.scores(users.user_emb[b], users.user_feat[b], users.user_x[b])
        rp, sp = p.scores(users.user_emb[b], users.user_feat[b], users.user_x[b])
        assert (ra == rp).all() and (sa == sp).all()
    # hand example: 2 fields (V = 2, 3), ad 0 holds keys {0, 2, 3} (a tag field with two values),
    # ad 1 holds key 3 twice (binary L: once); user: field 1 values 0 and 1 -> keys 2, 3
    cards = np.array([2, 3], np.int32)
    w = np.array([1, 1, 0.5, 0.25, 9], np.float32)
    po = oracle.OraclePairs(np.zeros((2, 4), np.float32), np.array([0, 3, 5]), np.array([0, 2, 3, 3, 3], np.int32),
                            cards, w)
    uf = np.array([[-1, -1], [0, 1]], np.int32)
    ux = np.array([[0, 0], [2, 4]], np.float32)
    r, _ = po.scores(np.zeros(4, np.float32), uf, ux)
    assert (r == [0.5 * 2 + 0.25 * 4, 0.25 * 4]).all()
