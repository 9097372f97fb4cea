"""GPU parity of the batched tensor-core path (bf16, batch >= 16): tcgen05 GEMM + fused epilogue,
sampled exact threshold, candidate selection -- against the CPU oracle, and against the latency
path on the same inputs."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2511_22460_b200 import synth  # noqa: E402
from tests.test_gpu_parity import check_all, run  # noqa: E402


@pytest.fixture(scope="module")
def ebr():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_22460_b200 import ebr as m
    return m



@pytest.mark.parametrize("cfg,n,b,k", [("C3", 60_000, 40, 100),      # one group (pad 40 -> 64)
                                       ("C3", 45_000, 200, 64),      # two groups (128 + 72)
                                       ("C4", 90_001, 64, 300),      # d=64, F=64, alpha=1.2
                                       ("C5", 70_000, 16, 128)])     # smallest eligible batch
def test_batch_exact_bit_exact(ebr, cfg, n, b, k):
    inv, users = synth.make_config(cfg, mode="exact", n_ads=n, batch=b)
    idx = ebr.Index.of(inv)
    (ids, sc), ws = run(ebr, idx, users, k)
    assert check_all(oracle.Oracle.of(inv), users, ids, sc, k, "exact") == 0
    assert ebr.query_error(ws) == 0


@pytest.mark.parametrize("cfg,n,b,k", [("C3", 130_000, 130, 1000), ("C4", 100_000, 64, 1000)])
def test_batch_real_tolerance(ebr, cfg, n, b, k):
    inv, users = synth.make_config(cfg, mode="real", n_ads=n, batch=b)
    idx = ebr.Index.of(inv)
    (ids, sc), _ = run(ebr, idx, users, k)
    o = oracle.Oracle.of(inv)
    sel = list(range(0, b, max(1, b // 12)))      # a spread of users (full check is slow on CPU)
    sub = synth.Users(len(sel), users.slots, users.user_emb[sel], users.user_feat[sel], users.user_x[sel])
    check_all(o, sub, ids[sel], sc[sel], k, "real")


def test_batch_equals_latency_path(ebr):
    inv, users = synth.make_config("C3", mode="exact", n_ads=50_000, batch=48)
    idx = ebr.Index.of(inv)
    (ids_b, sc_b), _ = run(ebr, idx, users, 200)
    os.environ["EBR_NO_BATCH_PATH"] = "1"
    try:
        (ids_s, sc_s), _ = run(ebr, idx, users, 200)
    finally:
        del os.environ["EBR_NO_BATCH_PATH"]
    assert (ids_b == ids_s).all() and (sc_b == sc_s).all()


@pytest.mark.parametrize("b,env", [(200, {"EBR_PAIR": "0"}), (256, {"EBR_PAIR": "0"}),
                                   (256, {"EBR_DEEP_SMEM": "1"}), (96, {"EBR_DEEP_SMEM": "1"}),
                                   (256, {"EBR_PAIR": "0", "EBR_DEEP_SMEM": "1"})])
def test_kernel_variants_equal_default(ebr, b, env):
    """Two-group passes run the CTA-pair kernel (tcgen05.mma.cta_group::2, M = 256 users) by default;
    EBR_PAIR=0 selects the single-CTA kernel (two clustered CTAs, one M = 128 MMA each) and
    EBR_DEEP_SMEM=1 the users' deep operand in shared memory (SS MMA, three TMEM stages).  Every
    variant equals the oracle bit for bit in exact mode, hence the default."""
    inv, users = synth.make_config("C3", mode="exact", n_ads=70_000, batch=b)
    idx = ebr.Index.of(inv)
    (ids_p, sc_p), _ = run(ebr, idx, users, 150)
    os.environ.update(env)
    try:
        (ids_s, sc_s), ws = run(ebr, idx, users, 150)
    finally:
        for k_ in env:
            del os.environ[k_]
    assert (ids_p == ids_s).all() and (sc_p == sc_s).all()
    assert check_all(oracle.Oracle.of(inv), users, ids_s, sc_s, 150, "exact") == 0
    assert ebr.query_error(ws) == 0


def test_batch_overflow_falls_back_exactly(ebr):
    inv, users = synth.make_config("C3", mode="exact", n_ads=40_000, batch=20)
    idx = ebr.Index.of(inv)
    os.environ["EBR_TEST_CAND_CAP"] = "700"       # below the ~1 K candidates of a user: every user overflows
    try:
        (ids, sc), _ = run(ebr, idx, users, 100)
    finally:
        del os.environ["EBR_TEST_CAND_CAP"]
    assert check_all(oracle.Oracle.of(inv), users, ids, sc, 100, "exact") == 0


def test_batch_workspace_reuse_and_keys(ebr):
    inv, users = synth.make_config("C3", mode="exact", n_ads=40_000, batch=32)
    idx = ebr.Index.of(inv)
    ws = ebr.new_workspace(idx, 32, users.slots, 80)
    dev = torch.device("cuda")
    o = oracle.Oracle.of(inv)
    for trial in range(3):
        u2 = synth.make_users(inv, 32, mode="exact", seed=50 + trial)
        emb = torch.from_numpy(u2.user_emb.view(np.int16)).to(dev)
        feat = torch.from_numpy(u2.user_feat).to(dev)
        x = torch.from_numpy(u2.user_x).to(dev)
        ids = torch.empty((32, 80), dtype=torch.int32, device=dev)
        sc = torch.empty((32, 80), dtype=torch.float32, device=dev)
        ebr.score_topk(idx, emb, feat, x, 80, ids, sc, ws)
        torch.cuda.synchronize()
        assert check_all(o, u2, ids.cpu().numpy(), sc.cpu().numpy(), 80, "exact") == 0


@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_full_size_sampled_users(ebr, cfg):
    """BASELINE.json configs 3 and 4 at full size and batch, in bench.py's launch configuration
    (one call for the whole batch); a few users are checked against the oracle's full scoring
    and brute-force sort (the oracle finishes one 10M-ad user in seconds)."""
    c = synth.CONFIGS[cfg]
    inv, users = synth.make_config(cfg, mode="real")
    idx = ebr.Index.of(inv)
    (ids, sc), _ = run(ebr, idx, users, c.k)
    o = oracle.Oracle.of(inv)
    sel = [0, users.batch // 2, users.batch - 1]
    sub = synth.Users(len(sel), users.slots, users.user_emb[sel], users.user_feat[sel], users.user_x[sel])
    check_all(o, sub, ids[sel], sc[sel], c.k, "real")
    # every user: ids unique, inside the inventory, scores sorted
    assert ((ids >= 0) & (ids < inv.n_ads)).all()
    assert all(len(np.unique(r)) == c.k for r in ids)
    assert (np.diff(sc, axis=1) <= 0).all()


# ---- hot keys: one-hot columns of L (bit masks expanded on chip) on the tensor cores (R22) ----

def test_hot_columns_built(ebr):
    inv, _ = synth.make_config("C3", mode="exact", n_ads=60_000, batch=16)
    st = ebr.Index.of(inv).stats()
    assert st["n_hot"] > 0 and st["n_hot"] % 64 == 0
    assert 0 < st["hot_nnz"] <= st["nnz"]
    assert st["hot_bytes"] == 16 * ((inv.n_ads + 127) // 128 * 128)     # one 128-bit mask per ad
    inv32, _ = synth.make_config("C2", mode="exact", n_ads=20_000, batch=1)
    assert ebr.Index.of(inv32).stats()["n_hot"] == 0          # fp32 indexes never take the batched path


@pytest.mark.parametrize("cfg,n,b,k", [("C3", 70_000, 48, 150), ("C4", 60_000, 64, 400)])
def test_batch_hot_equals_cold(ebr, cfg, n, b, k):
    """exact mode: the hot columns (tensor cores) and the compressed lists (shared-memory
    scatter) give bit-identical top-K ids and scores."""
    inv, users = synth.make_config(cfg, mode="exact", n_ads=n, batch=b)
    idx = ebr.Index.of(inv)
    assert idx.stats()["n_hot"] > 0
    (ids_h, sc_h), _ = run(ebr, idx, users, k)
    os.environ["EBR_NO_HOT"] = "1"
    try:
        (ids_c, sc_c), _ = run(ebr, idx, users, k)
    finally:
        del os.environ["EBR_NO_HOT"]
    assert (ids_h == ids_c).all() and (sc_h == sc_c).all()
    assert check_all(oracle.Oracle.of(inv), users, ids_h, sc_h, k, "exact") == 0


def test_batch_hot_duplicate_slots(ebr):
    """R3: the same (field, value) twice in one user adds twice -- also when the key is hot."""
    inv, users = synth.make_config("C3", mode="exact", n_ads=50_000, batch=24)
    uf = users.user_feat.copy()
    ux = users.user_x.copy()
    uf[:, :4, 1] = uf[:, :4, 0]                   # low-cardinality fields: hot keys
    ux[:, :4, 1] = np.where(uf[:, :4, 1] >= 0, 0.5, 0.0).astype(np.float32)
    users = synth.Users(users.batch, users.slots, users.user_emb, uf, ux)
    idx = ebr.Index.of(inv)
    (ids, sc), _ = run(ebr, idx, users, 100)
    assert check_all(oracle.Oracle.of(inv), users, ids, sc, 100, "exact") == 0


def test_batch_without_hot_columns(ebr):
    """EBR_HOT_KEYS=0 at build: no dense columns, every key through the compressed lists."""
    os.environ["EBR_HOT_KEYS"] = "0"
    try:
        inv, users = synth.make_config("C4", mode="exact", n_ads=40_000, batch=20)
        idx = ebr.Index.of(inv)
    finally:
        del os.environ["EBR_HOT_KEYS"]
    assert idx.stats()["n_hot"] == 0
    (ids, sc), _ = run(ebr, idx, users, 120)
    assert check_all(oracle.Oracle.of(inv), users, ids, sc, 120, "exact") == 0


def test_batch_small_batch_large_inventory(ebr):
    """B = 4 on a >= 2^21-ad bf16 inventory takes the tensor-core path (one hot K block): exact."""
    inv, users = synth.make_config("C3", mode="exact", n_ads=2_200_000, batch=4)
    idx = ebr.Index.of(inv)
    assert idx.query_launches(4, users.slots, 100) != 1      # not the single latency-path launch
    (ids, sc), ws = run(ebr, idx, users, 100)
    assert check_all(oracle.Oracle.of(inv), users, ids, sc, 100, "exact") == 0
    assert ebr.query_error(ws) == 0


@pytest.mark.parametrize("G", [2, 4])
def test_batch_sharded_merge_equals_single(ebr, G):
    """A7 over the tensor-core path: each ad-range shard (own hot columns, own encoded lists)
    emits kappa keys, the merge of the G lists equals the one-index answer bit for bit."""
    inv, users = synth.make_config("C3", mode="exact", n_ads=160_000, batch=40)
    k = 150
    (ids1, sc1), _ = run(ebr, ebr.Index.of(inv), users, k)
    bounds = (np.linspace(0, inv.n_ads, G + 1) // 128 * 128).astype(int)
    bounds[-1] = inv.n_ads
    parts = []
    for g in range(G):
        idx = ebr.Index.of(inv, lo=bounds[g], hi=bounds[g + 1])
        assert idx.query_launches(40, users.slots, k) != 10      # the batched path on every shard
        keys, _ = run(ebr, idx, users, k, keys=True)
        parts.append(keys)
    gathered = torch.from_numpy(np.stack(parts).view(np.int64)).cuda()
    ids = torch.empty((40, k), dtype=torch.int32, device="cuda")
    sc = torch.empty((40, k), dtype=torch.float32, device="cuda")
    ebr.merge_topk(gathered, G, 40, k, ids, sc)
    torch.cuda.synchronize()
    assert (ids.cpu().numpy() == ids1).all() and (sc.cpu().numpy() == sc1).all()
    assert check_all(oracle.Oracle.of(inv), users, ids1, sc1, k, "exact") == 0


def test_batch_theta_rank_shortfall_reruns_exactly(ebr):
    """theta taken at a sample rank far below K leaves users with fewer than K candidates: the
    group is rerun at rank K and the answer stays exact."""
    inv, users = synth.make_config("C3", mode="exact", n_ads=60_000, batch=24)
    idx = ebr.Index.of(inv)
    os.environ["EBR_THETA_RANK"] = "1"
    try:
        (ids, sc), _ = run(ebr, idx, users, 200)
    finally:
        del os.environ["EBR_THETA_RANK"]
    assert check_all(oracle.Oracle.of(inv), users, ids, sc, 200, "exact") == 0
