"""NEXT-3 ablation parity: the paper's own inverted list (Alg. 1) queried by
Alg. 2 (l.346-364) on the GPU, and the same algorithm on this library's chunk codec, both equal the
oracle's wide term (scorer B, explicit feature-pair enumeration) for every ad -- bit for bit
in exact mode (dyadic weights: every fp32 partial sum is exact, so the AtomicAdd order does not
matter), within 1e-5 x sigma in real mode.  Layout edge cases: a full 256-ad block (group 8),
single-ad blocks (group 0), the padding lanes of Alg. 1 ("pad ls with 0") never adding to ad
h*256 + 0 (reading R5), duplicate query keys (additive, R3), keys without postings."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2511_22460_b200 import synth  # noqa: E402


@pytest.fixture(scope="module")
def ebr():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_22460_b200 import ebr as m
    return m


def items_of(inv, uf, ux):
    """The user's (key, w~) query items (Alg. 2 input): key = base_f + v, w~ = fl32(w x)."""
    base = np.concatenate([[0], np.cumsum(inv.field_card)[:-1]]).astype(np.int64)
    keys, w = [], []
    F, S = uf.shape
    for f in range(F):
        for s in range(S):
            v = uf[f, s]
            if v >= 0:
                keys.append(base[f] + v)
                w.append(np.float32(inv.cross_w[base[f] + v]) * np.float32(ux[f, s]))
    return np.array(keys, np.int32), np.array(w, np.float32)


def both(ebr, inv, keys, w):
    dev = torch.device("cuda")
    idx = ebr.Index.of(inv)
    pidx = ebr.PaperIndex(inv.ad_feat, inv.field_card)
    k = torch.from_numpy(keys).to(dev)
    ww = torch.from_numpy(w).to(dev)
    sp = torch.empty(inv.n_ads, dtype=torch.float32, device=dev)
    sc = torch.empty(inv.n_ads, dtype=torch.float32, device=dev)
    ebr.paper_hitmatch(pidx, k, ww, sp)
    ebr.chunk_hitmatch(idx, k, ww, sc)
    torch.cuda.synchronize()
    return sp.cpu().numpy().astype(np.float64), sc.cpu().numpy().astype(np.float64), pidx


@pytest.mark.parametrize("cfg,n,mode", [("C2", 200_000, "exact"), ("C1", 10_000, "exact"),
                                        ("C4", 150_001, "exact"), ("C2", 300_000, "real")])
def test_paper_and_chunk_hitmatch_equal_oracle(ebr, cfg, n, mode):
    inv, users = synth.make_config(cfg, mode=mode, n_ads=n, batch=3)
    o = oracle.Oracle.of(inv)
    for b in range(users.batch):
        keys, w = items_of(inv, users.user_feat[b], users.user_x[b])
        sp, sc, pidx = both(ebr, inv, keys, w)
        ref = o.wide_pairs(users.user_feat[b], users.user_x[b])
        if mode == "exact":
            assert (sp == ref).all() and (sc == ref).all()
        else:
            # sigma of the wide term = sum of |w~| over the ad's hits (R12)
            absw = np.abs(w)
            sig = np.zeros(inv.n_ads)
            base = np.concatenate([[0], np.cumsum(inv.field_card)[:-1]]).astype(np.int64)
            af = inv.ad_feat.astype(np.int64)
            for kk, aw in zip(keys, absw):
                f = int(np.searchsorted(base, kk, side="right") - 1)
                sig[af[:, f] == kk - base[f]] += aw
            tol = 1e-5 * sig + 1e-30
            assert (np.abs(sp - ref) <= tol).all() and (np.abs(sc - ref) <= tol).all()
    info = pidx.info()
    assert sum(info["blocks_per_group"]) > 0 and info["bytes"] > 0


def test_paper_layout_edge_cases(ebr):
    # field 0: value 0 on ads 0..255 (one full block, group 8) and on ad 261 (a single-ad block,
    # group 0); field 1: value 1 on ads 256, 300 and 310 (a 3-ad block in group 2, padded to 4 with
    # a 0 residual that must not add to ad 256 a second time); value 2 of field 1 has no posting
    n = 600
    feat = np.full((n, 2), -1, np.int32)
    feat[:256, 0] = 0
    feat[261, 0] = 0
    feat[256, 1] = 1
    feat[300, 1] = 1
    feat[310, 1] = 1
    cards = np.array([4, 3], np.int32)
    w = np.array([0.5, 0.25, 1.0, 2.0, 0.125, 4.0, 8.0], np.float32)
    inv = synth.Inventory(n, 16, "f32", np.zeros((n, 16), np.float32), feat, cards, w, 0)
    keys = np.array([0, 5, 6, 5, 99999], np.int32)        # key 5 twice (additive), 6 empty, 99999 invalid
    wq = np.array([0.5, 0.25, 3.0, 0.125, 7.0], np.float32)
    sp, sc, pidx = both(ebr, inv, keys, wq)
    ref = np.zeros(n)
    ref[:256] += 0.5
    ref[261] += 0.5
    ref[256] += 0.375
    ref[300] += 0.375
    ref[310] += 0.375
    assert (sp == ref).all() and (sc == ref).all()
    blocks = pidx.info()["blocks_per_group"]
    assert blocks[8] == 1 and blocks[0] == 1 and blocks[2] == 1
