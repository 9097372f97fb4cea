"""GPU parity where the north star's targets live (BASELINE.json configs at full size, and the
large-K paths): the CUDA path through the C-ABI against the CPU oracle, element by element.

  * batched path (tcgen05) at K = 4096 and 10 000 -- final_kernel's global-memory select (more
    candidates than its shared-memory buffer) and theta's rank-K rerun selecting from global memory;
  * latency path at K = 4096 and 10 000 on >= 3 M ads (B = 1 and 3);
  * C3 at full size (10 M ads, B = 256, K = 1000): 32 seeded users in real mode, 8 users bit-exact
    in exact mode; C4 at full size with all 64 users; one C5 point (20 M ads, B = 1024, K = 10 000)
    on 3 users -- every call in bench.py's launch configuration (one call for the whole batch);
  * a CUDA-graph capture of a batched call replays to the same output as the direct call (the
    batched path enqueues without host synchronisation, include/ebr.h).

Scores: Eq. 9; top k (l.157); ties by ascending id (reading R13)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2511_22460_b200 import synth  # noqa: E402
from tests.parity import check_many  # noqa: E402
from tests.test_gpu_parity import run  # noqa: E402


@pytest.fixture(scope="module")
def ebr():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_22460_b200 import ebr as m
    return m


def batched(idx, users, k):
    B, _, S = users.user_feat.shape
    return idx.query_launches(B, S, k) != (B + 3) // 4


def sanity(ids, sc, n, k):
    """every user: ids unique and inside the inventory, scores sorted descending"""
    kk = min(k, n)
    assert ((ids[:, :kk] >= 0) & (ids[:, :kk] < n)).all()
    assert all(len(np.unique(r[:kk])) == kk for r in ids)
    assert (np.diff(sc[:, :kk], axis=1) <= 0).all()


# ------------------------------------------------------------------ large K, batched path

@pytest.mark.parametrize("k", [4096, 10000])
def test_batched_large_k_exact(ebr, k):
    inv, users = synth.make_config("C3", mode="exact", n_ads=700_000, batch=24)
    idx = ebr.Index.of(inv)
    assert batched(idx, users, k)
    (ids, sc), ws = run(ebr, idx, users, k)
    assert check_many(oracle.Oracle.of(inv), users, ids, sc, k, "exact") == 0
    assert ebr.query_error(ws) == 0


@pytest.mark.parametrize("k", [4096, 10000])
def test_batched_large_k_rank_rerun(ebr, k):
    """theta taken at sample rank 1: every user is short of K candidates, so the gated rerun
    takes theta at rank K of the sample (a buffer larger than theta's shared memory)."""
    inv, users = synth.make_config("C3", mode="exact", n_ads=700_000, batch=20, seed_offset=1)
    idx = ebr.Index.of(inv)
    os.environ["EBR_THETA_RANK"] = "1"
    try:
        (ids, sc), _ = run(ebr, idx, users, k)
    finally:
        del os.environ["EBR_THETA_RANK"]
    assert check_many(oracle.Oracle.of(inv), users, ids, sc, k, "exact") == 0


def test_batched_large_k_real(ebr):
    inv, users = synth.make_config("C3", mode="real", n_ads=800_000, batch=40)
    idx = ebr.Index.of(inv)
    (ids, sc), _ = run(ebr, idx, users, 10000)
    check_many(oracle.Oracle.of(inv), users, ids, sc, 10000, "real", sel=range(0, 40, 3))


# ------------------------------------------------------------------ large K, latency path

@pytest.mark.parametrize("cfg,b,k", [("C2", 1, 4096), ("C2", 1, 10000), ("C2", 3, 10000), ("C5", 1, 10000)])
def test_latency_large_k_exact(ebr, cfg, b, k):
    inv, users = synth.make_config(cfg, mode="exact", n_ads=3_000_000, batch=b)
    idx = ebr.Index.of(inv)
    assert not batched(idx, users, k)
    (ids, sc), ws = run(ebr, idx, users, k)
    assert check_many(oracle.Oracle.of(inv), users, ids, sc, k, "exact") == 0
    assert ebr.query_error(ws) == 0


# ------------------------------------------------------------------ BASELINE configs at full size

def test_full_c3_real_32_users(ebr):
    c = synth.CONFIGS["C3"]
    inv, users = synth.make_config("C3", mode="real")
    idx = ebr.Index.of(inv)
    assert batched(idx, users, c.k)
    (ids, sc), _ = run(ebr, idx, users, c.k)
    sel = np.random.default_rng(3).choice(users.batch, 32, replace=False)
    check_many(oracle.Oracle.of(inv), users, ids, sc, c.k, "real", sel=sel)
    sanity(ids, sc, inv.n_ads, c.k)


def test_full_c3_exact_bit_exact(ebr):
    c = synth.CONFIGS["C3"]
    inv, users = synth.make_config("C3", mode="exact")
    idx = ebr.Index.of(inv)
    (ids, sc), ws = run(ebr, idx, users, c.k)
    sel = [0, 37, 64, 127, 128, 200, 254, 255]          # both 128-user groups, first and last
    assert check_many(oracle.Oracle.of(inv), users, ids, sc, c.k, "exact", sel=sel) == 0
    assert ebr.query_error(ws) == 0
    sanity(ids, sc, inv.n_ads, c.k)


def test_full_c4_all_users(ebr):
    c = synth.CONFIGS["C4"]
    inv, users = synth.make_config("C4", mode="real")
    idx = ebr.Index.of(inv)
    assert batched(idx, users, c.k)
    (ids, sc), _ = run(ebr, idx, users, c.k)
    check_many(oracle.Oracle.of(inv), users, ids, sc, c.k, "real")


def test_c5_point_b1024_k10000(ebr):
    inv, users = synth.make_config("C5", mode="real", batch=1024)
    idx = ebr.Index.of(inv)
    k = 10000
    assert batched(idx, users, k)
    (ids, sc), ws = run(ebr, idx, users, k)
    check_many(oracle.Oracle.of(inv), users, ids, sc, k, "real", sel=[0, 511, 1023])
    sanity(ids, sc, inv.n_ads, k)
    assert ebr.query_error(ws) == 0


# ------------------------------------------------------------------ graph capture (async boundary)

def test_batched_call_graph_capture(ebr):
    inv, users = synth.make_config("C3", mode="exact", n_ads=300_000, batch=160)
    idx = ebr.Index.of(inv)
    k = 500
    assert batched(idx, users, k)
    dev = torch.device("cuda")
    emb = torch.from_numpy(users.user_emb.view(np.int16)).to(dev)
    feat = torch.from_numpy(users.user_feat).to(dev)
    x = torch.from_numpy(users.user_x).to(dev)
    ws = ebr.new_workspace(idx, users.batch, users.slots, k)
    outs = [(torch.full((users.batch, k), -7, dtype=torch.int32, device=dev),
             torch.zeros((users.batch, k), dtype=torch.float32, device=dev)) for _ in range(2)]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ebr.score_topk(idx, emb, feat, x, k, outs[0][0], outs[0][1], ws, st)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        ebr.score_topk(idx, emb, feat, x, k, outs[1][0], outs[1][1], ws, st)
    for _ in range(3):
        outs[1][0].fill_(-7)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    ids, sc = outs[1][0].cpu().numpy(), outs[1][1].cpu().numpy()
    assert check_many(oracle.Oracle.of(inv), users, ids, sc, k, "exact", sel=[0, 80, 159]) == 0
