"""Device-side index build (Alg. 1): the inverted list
built by GPU kernels is bit-identical to the host encoder's (every exported array), its decoded
lists equal the oracle's postings (keys = feature indices, values = ad ids), queries on it
equal queries on the host-built index, bounds errors are detected on the device, and an index can
be rebuilt and swapped while queries on the old one are in flight (double-buffered refresh)."""
import time

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


@pytest.mark.parametrize("cfg,n", [("C1", 10_000), ("C2", 300_000), ("C3", 400_000), ("C4", 200_001), ("C1", 1)])
def test_device_build_bit_identical(ebr, cfg, n):
    inv, _ = synth.make_config(cfg, mode="real", n_ads=n, batch=1)
    h = ebr.Index.of(inv)
    d = ebr.Index.of(inv, device_build=True)
    for which in range(6):
        a, b = h.export(which), d.export(which)
        assert a.shape == b.shape and (a == b).all(), which
    sh, sd = h.stats(), d.stats()
    for k in ("nnz", "chunks", "payload_words", "index_bytes", "n_hot", "hot_nnz"):
        assert sh[k] == sd[k], k
    # decoded lists == the oracle's postings (a spread of keys incl. the longest)
    off, ads = oracle.Oracle.of(inv).postings()
    lens = np.diff(off)
    M = len(lens)
    for key in list(np.argsort(-lens)[:5]) + list(range(0, M, max(1, M // 50))):
        assert (d.debug_decode(int(key)) == ads[off[key]:off[key + 1]]).all()


def test_device_build_query_parity_and_shards(ebr):
    inv, users = synth.make_config("C3", mode="exact", n_ads=150_000, batch=40)
    o = oracle.Oracle.of(inv)
    d = ebr.Index.of(inv, device_build=True)
    (ids, sc), _ = run(ebr, d, users, 300)
    assert check_many(o, users, ids, sc, 300, "exact") == 0
    # a shard (ad_begin > 0) built on the device equals the host-built shard
    a = ebr.Index.of(inv, lo=50_048, hi=100_000)
    b = ebr.Index.of(inv, lo=50_048, hi=100_000, device_build=True)
    for which in range(6):
        assert (a.export(which) == b.export(which)).all(), which


def test_device_build_rejects_bad_values(ebr):
    inv, _ = synth.make_config("C1", mode="real", n_ads=5000, batch=1)
    feat = inv.ad_feat.copy()
    feat[1234, 3] = inv.field_card[3]
    with pytest.raises(ebr.EbrError):
        ebr.Index(inv.ad_emb, feat, inv.field_card, inv.cross_w, device_build=True)
    feat[1234, 3] = -2
    with pytest.raises(ebr.EbrError):
        ebr.Index(inv.ad_emb, feat, inv.field_card, inv.cross_w, device_build=True)


def test_refresh_while_queries_in_flight(ebr):
    """Queries on index X are enqueued on stream Q; index Y (the refreshed inventory) is built on
    another stream meanwhile and swapped in; results of both match their own oracle."""
    inv_x, users = synth.make_config("C3", mode="exact", n_ads=300_000, batch=32)
    inv_y, _ = synth.make_config("C3", mode="exact", n_ads=300_000, batch=32, seed_offset=3)
    k = 200
    dev = torch.device("cuda")
    x = ebr.Index.of(inv_x, device_build=True)
    emb = torch.from_numpy(users.user_emb.view(np.int16)).to(dev)
    feat = torch.from_numpy(users.user_feat).to(dev)
    ux = torch.from_numpy(users.user_x).to(dev)
    ws = ebr.new_workspace(x, users.batch, users.slots, k)
    q = torch.cuda.Stream()
    outs_x = []
    for _ in range(8):
        ids = torch.empty((users.batch, k), dtype=torch.int32, device=dev)
        sc = torch.empty((users.batch, k), dtype=torch.float32, device=dev)
        ebr.score_topk(x, emb, feat, ux, k, ids, sc, ws, q)
        outs_x.append((ids, sc))
    t0 = time.perf_counter()
    y = ebr.Index.of(inv_y, device_build=True)
    build_s = time.perf_counter() - t0
    ws_y = ebr.new_workspace(y, users.batch, users.slots, k)
    ids_y = torch.empty((users.batch, k), dtype=torch.int32, device=dev)
    sc_y = torch.empty((users.batch, k), dtype=torch.float32, device=dev)
    ebr.score_topk(y, emb, feat, ux, k, ids_y, sc_y, ws_y, q)      # the swap: new queries use Y
    q.synchronize()
    x.close()                                                    # the old index, after its queries
    ox, oy = oracle.Oracle.of(inv_x), oracle.Oracle.of(inv_y)
    ref = outs_x[0]
    assert check_many(ox, users, ref[0].cpu().numpy(), ref[1].cpu().numpy(), k, "exact", sel=[0, 13, 31]) == 0
    for ids, sc in outs_x[1:]:
        assert torch.equal(ids, ref[0]) and torch.equal(sc, ref[1])
    assert check_many(oy, users, ids_y.cpu().numpy(), sc_y.cpu().numpy(), k, "exact", sel=[0, 13, 31]) == 0
    assert build_s < 60
