"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Bit-exact for integer work (decoded posting lists, top-K ids in exact mode), tolerance for fp
(1e-5 * sigma, tests/parity.py).  Sizes span several ranges/tiles with ragged tails; the full
C1 and C2 configs run at their BASELINE.json sizes in the launch configuration bench.py uses."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2511_22460_b200 import synth  # noqa: E402
from tests.parity import check_user  # noqa: E402


@pytest.fixture(scope="module")
def ebr():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_22460_b200 import ebr as m
    return m


def run(ebr, idx, users, k, keys=False, stream=None):
    dev = torch.device("cuda", idx.device)
    B, F, S = users.user_feat.shape
    emb = torch.from_numpy(np.ascontiguousarray(users.user_emb).view(
        np.int16 if users.user_emb.dtype == np.uint16 else np.float32)).to(dev)
    feat = torch.from_numpy(users.user_feat).to(dev)
    x = torch.from_numpy(users.user_x).to(dev)
    ws = ebr.new_workspace(idx, B, S, k)
    if keys:
        out = torch.empty((B, k), dtype=torch.int64, device=dev)
        ebr.score_topk_keys(idx, emb, feat, x, k, out, ws, stream)
        torch.cuda.synchronize()
        return out.cpu().numpy().view(np.uint64), ws
    ids = torch.empty((B, k), dtype=torch.int32, device=dev)
    sc = torch.empty((B, k), dtype=torch.float32, device=dev)
    ebr.score_topk(idx, emb, feat, x, k, ids, sc, ws, stream)
    torch.cuda.synchronize()
    return (ids.cpu().numpy(), sc.cpu().numpy()), ws


def check_all(o, users, ids, sc, k, mode, id_base=0):
    mism = 0
    for b in range(users.batch):
        r, s = o.scores(users.user_emb[b], users.user_feat[b], users.user_x[b])
        mism += check_user(ids[b], sc[b], r, s, k, mode, id_base=id_base)
    return mism


# ---------------------------------------------------------------- A0/A2: decode(encode(L)) == L

def test_device_decode_equals_postings(ebr):
    inv = synth.make_inventory(70_000, 8, 12, alpha=1.2, seed=21)
    idx = ebr.Index.of(inv)
    off, ads = oracle.Oracle.of(inv).postings()
    rng = np.random.default_rng(0)
    keys = np.concatenate([np.arange(0, min(400, idx.n_keys)),
                           np.argsort(-np.diff(off))[:50],                 # the hottest lists
                           rng.integers(0, idx.n_keys, 300)])
    for k in np.unique(keys):
        got = idx.debug_decode(int(k))
        assert (got == ads[off[k]:off[k + 1]]).all(), k
    st = idx.stats()
    assert st["nnz"] == off[-1] and st["n_ads"] == inv.n_ads


# ---------------------------------------------------------------- exact mode: bit-exact top-K

@pytest.mark.parametrize("cfg,n,b,k", [("C1", 10_000, 1, 100), ("C1", 10_000, 3, 100),
                                       ("C1", 9_973, 8, 257), ("C2", 200_003, 2, 500),
                                       ("C4", 50_001, 5, 1000), ("C3", 40_000, 8, 1000)])
def test_exact_mode_bit_exact(ebr, cfg, n, b, k):
    inv, users = synth.make_config(cfg, mode="exact", n_ads=n, batch=b)
    idx = ebr.Index.of(inv)
    (ids, sc), ws = run(ebr, idx, users, k)
    assert check_all(oracle.Oracle.of(inv), users, ids, sc, k, "exact") == 0
    assert ebr.query_error(ws) == 0


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("d", [16, 64, 100, 128, 200])
def test_exact_mode_widths(ebr, dtype, d):
    inv = synth.make_inventory(5_000, d, 6, dtype=dtype, mode="exact", seed=d)
    users = synth.make_users(inv, 3, mode="exact", seed=d + 1)
    idx = ebr.Index.of(inv)
    (ids, sc), _ = run(ebr, idx, users, 64)
    assert check_all(oracle.Oracle.of(inv), users, ids, sc, 64, "exact") == 0


# ---------------------------------------------------------------- real mode: tolerance

@pytest.mark.parametrize("cfg,n,b,k", [("C1", 10_000, 1, 100), ("C2", 300_000, 4, 500),
                                       ("C3", 60_000, 8, 1000), ("C4", 80_000, 3, 1000)])
def test_real_mode_tolerance(ebr, cfg, n, b, k):
    inv, users = synth.make_config(cfg, mode="real", n_ads=n, batch=b)
    idx = ebr.Index.of(inv)
    (ids, sc), _ = run(ebr, idx, users, k)
    check_all(oracle.Oracle.of(inv), users, ids, sc, k, "real")


def test_full_c1_and_c2(ebr):
    """BASELINE.json configs 1 and 2 at full size, in bench.py's launch configuration."""
    for cfg in ("C1", "C2"):
        c = synth.CONFIGS[cfg]
        for mode in ("exact", "real"):
            inv, users = synth.make_config(cfg, mode=mode)
            idx = ebr.Index.of(inv)
            (ids, sc), _ = run(ebr, idx, users, c.k)
            check_all(oracle.Oracle.of(inv), users, ids, sc, c.k, mode)
            del idx


def test_bf16_quantisation_vs_fp32_masters(ebr):
    """bf16 path vs the oracle on fp32 master embeddings: 2e-3 * sigma (north star)."""
    inv32, users32 = synth.make_config("C1", mode="real", n_ads=20_000, batch=2)
    inv16 = synth.Inventory(inv32.n_ads, inv32.d, "bf16", synth.f32_to_bf16_bits(inv32.ad_emb),
                            inv32.ad_feat, inv32.field_card, inv32.cross_w)
    users16 = synth.Users(2, users32.slots, synth.f32_to_bf16_bits(users32.user_emb),
                          users32.user_feat, users32.user_x)
    (ids, sc), _ = run(ebr, ebr.Index.of(inv16), users16, 50)
    o = oracle.Oracle.of(inv32)
    for b in range(2):
        r, s = o.scores(users32.user_emb[b], users32.user_feat[b], users32.user_x[b])
        assert (np.abs(sc[b] - r[ids[b]]) <= 2e-3 * s[ids[b]]).all()


# ---------------------------------------------------------------- edge cases

def test_k_larger_than_inventory_and_k1(ebr):
    inv, users = synth.make_config("C1", mode="exact", n_ads=300, batch=2)
    idx = ebr.Index.of(inv)
    o = oracle.Oracle.of(inv)
    for k in (1, 299, 300, 301, 1000):
        (ids, sc), _ = run(ebr, idx, users, k)
        assert check_all(o, users, ids, sc, k, "exact") == 0


def test_tiny_inventories(ebr):
    for n in (1, 2, 31, 33, 127, 129):
        inv, users = synth.make_config("C1", mode="exact", n_ads=n, batch=2)
        idx = ebr.Index.of(inv)
        (ids, sc), _ = run(ebr, idx, users, 5)
        assert check_all(oracle.Oracle.of(inv), users, ids, sc, 5, "exact") == 0


def test_empty_users_and_zero_embeddings(ebr):
    # zero-feature users == plain dual tower; zero embeddings == scorer B (pair enumeration)
    inv, users = synth.make_config("C1", mode="exact", n_ads=4_000, batch=2)
    users.user_feat[0] = -1
    users.user_x[0] = 0
    inv0 = synth.Inventory(inv.n_ads, inv.d, inv.dtype, np.zeros_like(inv.ad_emb), inv.ad_feat,
                           inv.field_card, inv.cross_w)
    o = oracle.Oracle.of(inv)
    (ids, sc), _ = run(ebr, ebr.Index.of(inv), users, 40)
    assert check_all(o, users, ids, sc, 40, "exact") == 0
    (ids0, sc0), _ = run(ebr, ebr.Index.of(inv0), users, 4000)
    wide = o.wide_pairs(users.user_feat[1], users.user_x[1])
    order = np.lexsort((np.arange(inv.n_ads), -wide))
    assert (ids0[1] == order).all() and (sc0[1] == wide[order]).all()


def test_all_ties(ebr):
    inv = synth.make_inventory(3_000, 8, 2, mode="exact", seed=4)
    inv.ad_emb[:] = 0
    inv.ad_feat[:] = -1
    users = synth.make_users(inv, 2, mode="exact", seed=5)
    (ids, sc), _ = run(ebr, ebr.Index.of(inv), users, 100)
    assert (ids == np.arange(100)).all() and (sc == 0).all()


def test_bad_user_value_raises_flag(ebr):
    inv, users = synth.make_config("C1", mode="exact", n_ads=2_000, batch=1)
    users.user_feat[0, 0, 0] = inv.field_card[0] + 5
    (ids, sc), ws = run(ebr, ebr.Index.of(inv), users, 10)
    assert ebr.query_error(ws) == 1
    assert ebr.query_error(ws) == 0          # cleared


@pytest.mark.parametrize("b", [1, 40])
def test_negative_user_value_raises_flag(ebr, b):
    """A user value below -1 is outside [-1, V_f): skipped (as if empty) and flagged (ebr.h), on
    the latency path (b=1) and the batched path (b=40, bf16)."""
    cfg = "C1" if b == 1 else "C3"
    inv, users = synth.make_config(cfg, mode="exact", n_ads=80_000, batch=b)
    users.user_feat[0, 0, 0] = -5
    (ids, sc), ws = run(ebr, ebr.Index.of(inv), users, 50)
    assert ebr.query_error(ws) == 1
    users.user_feat[0, 0, 0] = -1
    assert check_all(oracle.Oracle.of(inv), users, ids, sc, 50, "exact") == 0


def test_workspace_reuse_across_indexes(ebr):
    """One workspace serves successive indexes of the same geometry (state left clean)."""
    inv, users = synth.make_config("C1", mode="exact", n_ads=5_000, batch=3)
    idx = ebr.Index.of(inv)
    ws = ebr.new_workspace(idx, 3, users.slots, 50)
    o = oracle.Oracle.of(inv)
    dev = torch.device("cuda")
    for trial in range(3):
        users2 = synth.make_users(inv, 3, mode="exact", seed=100 + trial)
        ids = torch.empty((3, 50), dtype=torch.int32, device=dev)
        sc = torch.empty((3, 50), dtype=torch.float32, device=dev)
        ebr.score_topk(idx, torch.from_numpy(users2.user_emb).to(dev), torch.from_numpy(users2.user_feat).to(dev),
                       torch.from_numpy(users2.user_x).to(dev), 50, ids, sc, ws)
        torch.cuda.synchronize()
        assert check_all(o, users2, ids.cpu().numpy(), sc.cpu().numpy(), 50, "exact") == 0


def test_uninitialised_workspace_self_inits(ebr):
    inv, users = synth.make_config("C1", mode="exact", n_ads=3_000, batch=2)
    idx = ebr.Index.of(inv)
    ws = torch.full((idx.workspace_bytes(2, users.slots, 20),), 7, dtype=torch.uint8, device="cuda")
    dev = torch.device("cuda")
    ids = torch.empty((2, 20), dtype=torch.int32, device=dev)
    sc = torch.empty((2, 20), dtype=torch.float32, device=dev)
    ebr.score_topk(idx, torch.from_numpy(users.user_emb).to(dev), torch.from_numpy(users.user_feat).to(dev),
                   torch.from_numpy(users.user_x).to(dev), 20, ids, sc, ws)
    torch.cuda.synchronize()
    assert check_all(oracle.Oracle.of(inv), users, ids.cpu().numpy(), sc.cpu().numpy(), 20, "exact") == 0


def test_invalid_arguments(ebr):
    inv, users = synth.make_config("C1", mode="exact", n_ads=100, batch=1)
    idx = ebr.Index.of(inv)
    with pytest.raises(ebr.EbrError):
        run(ebr, idx, users, 0)
    with pytest.raises(ebr.EbrError):
        run(ebr, idx, users, ebr.MAX_K + 1)
    bad = inv.ad_feat.copy()
    bad[3, 1] = inv.field_card[1]
    with pytest.raises(ebr.EbrError):
        ebr.Index(inv.ad_emb, bad, inv.field_card, inv.cross_w)


# ---------------------------------------------------------------- host (e2e) variant, keys

def test_host_variant_equals_device(ebr):
    # exact mode: the real-mode wide sum order is not deterministic across runs (reading R9)
    inv, users = synth.make_config("C2", mode="exact", n_ads=100_000, batch=3)
    idx = ebr.Index.of(inv)
    (ids, sc), _ = run(ebr, idx, users, 200)
    ws = ebr.new_workspace(idx, 3, users.slots, 200, host=True)
    hid = np.empty((3, 200), np.int32)
    hsc = np.empty((3, 200), np.float32)
    ebr.score_topk_host(idx, users.user_emb, users.user_feat, users.user_x, 200, hid, hsc, ws)
    assert (hid == ids).all() and (hsc == sc).all()


def test_host_variant_staged_and_direct(ebr):
    """both copy strategies of ebr_score_topk_host: a small request (pinned staging, one H2D and
    one D2H) after a large one (> 1 MB of outputs: one copy per array), then small again"""
    inv, users = synth.make_config("C2", mode="exact", n_ads=100_000, batch=70)
    idx = ebr.Index.of(inv)
    for b, k in ((2, 50), (70, 2000), (5, 300)):
        sub = synth.Users(b, users.slots, users.user_emb[:b], users.user_feat[:b], users.user_x[:b])
        (ids, sc), _ = run(ebr, idx, sub, k)
        ws = ebr.new_workspace(idx, b, users.slots, k, host=True)
        hid = np.empty((b, k), np.int32)
        hsc = np.empty((b, k), np.float32)
        ebr.score_topk_host(idx, sub.user_emb, sub.user_feat, sub.user_x, k, hid, hsc, ws)
        assert (hid == ids).all() and (hsc == sc).all()


# ---------------------------------------------------------------- A7: shard + merge == 1 GPU

@pytest.mark.parametrize("G", [2, 3, 8])
def test_sharded_merge_equals_single(ebr, G):
    inv, users = synth.make_config("C1", mode="exact", n_ads=50_000, batch=4)
    k = 300
    (ids1, sc1), _ = run(ebr, ebr.Index.of(inv), users, k)
    bounds = np.linspace(0, inv.n_ads, G + 1).astype(int)
    parts = []
    for g in range(G):
        idx = ebr.Index.of(inv, lo=bounds[g], hi=bounds[g + 1])
        keys, _ = run(ebr, idx, users, k, keys=True)
        parts.append(keys)
    gathered = torch.from_numpy(np.stack(parts).view(np.int64)).cuda()
    ids = torch.empty((4, k), dtype=torch.int32, device="cuda")
    sc = torch.empty((4, k), dtype=torch.float32, device="cuda")
    ebr.merge_topk(gathered, G, 4, k, ids, sc)
    torch.cuda.synchronize()
    assert (ids.cpu().numpy() == ids1).all() and (sc.cpu().numpy() == sc1).all()
    assert check_all(oracle.Oracle.of(inv), users, ids1, sc1, k, "exact") == 0


def test_shard_smaller_than_k_pads(ebr):
    inv, users = synth.make_config("C1", mode="exact", n_ads=500, batch=2)
    k = 400
    parts = []
    for lo, hi in ((0, 100), (100, 500)):
        keys, _ = run(ebr, ebr.Index.of(inv, lo=lo, hi=hi), users, k, keys=True)
        parts.append(keys)
    assert (parts[0][:, 100:] == 0).all()
    gathered = torch.from_numpy(np.stack(parts).view(np.int64)).cuda()
    ids = torch.empty((2, k), dtype=torch.int32, device="cuda")
    sc = torch.empty((2, k), dtype=torch.float32, device="cuda")
    ebr.merge_topk(gathered, 2, 2, k, ids, sc)
    torch.cuda.synchronize()
    assert check_all(oracle.Oracle.of(inv), users, ids.cpu().numpy(), sc.cpu().numpy(), k, "exact") == 0


@pytest.mark.parametrize("G,n,k", [(2, 300, 400), (8, 8 * 600, 4096)])
def test_merge_total_below_k_pads(ebr, G, n, k):
    """All shards together hold fewer than K ads: the padding keys (0) must not displace real
    keys in the merge (the radix select needs unique keys; padding becomes distinct
    sentinels below every real kappa)."""
    inv, users = synth.make_config("C1", mode="exact", n_ads=n, batch=2)
    bounds = np.linspace(0, n, G + 1).astype(int)
    parts = []
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        keys, _ = run(ebr, ebr.Index.of(inv, lo=int(lo), hi=int(hi)), users, k, keys=True)
        parts.append(keys)
    gathered = torch.from_numpy(np.stack(parts).view(np.int64)).cuda()
    ids = torch.empty((2, k), dtype=torch.int32, device="cuda")
    sc = torch.empty((2, k), dtype=torch.float32, device="cuda")
    ebr.merge_topk(gathered, G, 2, k, ids, sc)
    torch.cuda.synchronize()
    ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
    assert (ids[:, n:] == -1).all() and np.isneginf(sc[:, n:]).all()
    assert check_all(oracle.Oracle.of(inv), users, ids, sc, k, "exact") == 0


@pytest.mark.parametrize("dtype,b", [("f32", 1), ("bf16", 3)])
def test_multi_tile_latency_path(ebr, dtype, b):
    """Inventories whose per-CTA range exceeds one shared-memory tile (N > 148 x 16384): the
    latency kernel loops over tiles and keeps fused scores in the L2 scratch."""
    inv = synth.make_inventory(3_000_001, 64, 12, dtype=dtype, mode="exact", seed=77)
    users = synth.make_users(inv, b, mode="exact", seed=78)
    idx = ebr.Index.of(inv)
    (ids, sc), _ = run(ebr, idx, users, 300)
    assert check_all(oracle.Oracle.of(inv), users, ids, sc, 300, "exact") == 0
