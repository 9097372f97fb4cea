"""NEXT-4, multi-valued ad fields (tags; reading R4): the index built on the device
from per-ad key lists (ebr_build_index_lists) equals the ad_feat build when every ad has one value
per field (every exported array bit for bit), and with several values per field the query paths
(latency, B = 2; batched tensor-core, B = 40) equal the oracle's scorer A on the same lists
(oracle_scores_user_pairs: Eq. 9 with L given by its nonzeros) bit for bit in exact mode.  A key
listed twice for one ad or outside [0, M) is rejected."""
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


def lists_of(inv, extra_fields=(), seed=0, max_extra=3):
    """per-ad global key lists: the ad's ad_feat values plus, for `extra_fields`, up to max_extra
    further distinct values drawn uniformly (tags)."""
    rng = np.random.default_rng(seed)
    base = np.concatenate([[0], np.cumsum(inv.field_card)[:-1]]).astype(np.int64)
    lists = []
    for a in range(inv.n_ads):
        ks = [int(base[f] + v) for f, v in enumerate(inv.ad_feat[a]) if v >= 0]
        for f in extra_fields:
            vals = set(int(x) for x in rng.integers(0, inv.field_card[f], rng.integers(0, max_extra + 1)))
            vals.discard(int(inv.ad_feat[a, f]))
            ks += [int(base[f] + v) for v in sorted(vals)]
        lists.append(ks)
    off = np.concatenate([[0], np.cumsum([len(k) for k in lists])]).astype(np.int64)
    keys = np.array([k for ks in lists for k in ks], np.int32)
    return off, keys


def test_lists_build_equals_ad_feat_build(ebr):
    inv, _ = synth.make_config("C3", mode="real", n_ads=120_000, batch=1)
    off, keys = lists_of(inv)
    a = ebr.Index.of(inv, device_build=True)
    b = ebr.Index.from_lists(inv.ad_emb, off, keys, inv.field_card, inv.cross_w)
    for which in range(6):
        assert (a.export(which) == b.export(which)).all(), which


@pytest.mark.parametrize("batch,k", [(2, 300), (40, 300)])
def test_multi_valued_fields_equal_oracle(ebr, batch, k):
    inv, users = synth.make_config("C3", mode="exact", n_ads=150_000, batch=batch)
    off, keys = lists_of(inv, extra_fields=(2, 4, 9), seed=batch)
    idx = ebr.Index.from_lists(inv.ad_emb, off, keys, inv.field_card, inv.cross_w)
    assert idx.stats()["nnz"] == len(keys)
    (ids, sc), ws = run(ebr, idx, users, k)
    o = oracle.OraclePairs(inv.ad_emb, off, keys, inv.field_card, inv.cross_w)
    assert check_many(o, users, ids, sc, k, "exact") == 0
    assert ebr.query_error(ws) == 0


def test_lists_reject_duplicates_and_bad_keys(ebr):
    inv, _ = synth.make_config("C1", mode="real", n_ads=2000, batch=1)
    off, keys = lists_of(inv)
    dup = keys.copy()
    dup[off[5] + 1] = dup[off[5]]                    # ad 5 lists one key twice
    with pytest.raises(ebr.EbrError):
        ebr.Index.from_lists(inv.ad_emb, off, dup, inv.field_card, inv.cross_w)
    bad = keys.copy()
    bad[7] = int(inv.field_card.sum())
    with pytest.raises(ebr.EbrError):
        ebr.Index.from_lists(inv.ad_emb, off, bad, inv.field_card, inv.cross_w)
