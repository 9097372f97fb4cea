"""NEXT-4, in-query IPNN (Eq. 7-8): ebr_ipnn_extend's h~ = [h, W u] against
the oracle's fp64 extension (fp32: within the fp32 summation bound; bf16: within one bf16 rounding
of it), and a full query whose users and ads were extended on the GPU against the oracle's scores
on the same extended vectors (Eq. 8: the deep term is then <h_u, h_a> + <W_u u, W_v v>)."""
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


def extend(ebr, h, u, W):
    dev = torch.device("cuda")
    th = torch.from_numpy(h.view(np.int16) if h.dtype == np.uint16 else h).to(dev)
    out = torch.empty((h.shape[0], h.shape[1] + W.shape[0]), dtype=th.dtype, device=dev)
    ebr.ipnn_extend(th, torch.from_numpy(u).to(dev), torch.from_numpy(W).to(dev), out)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    return o.view(np.uint16) if h.dtype == np.uint16 else o


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_ipnn_extend_equals_oracle(ebr, dtype):
    rng = np.random.default_rng(11)
    rows, d0, n, d1 = 3000, 96, 40, 32
    h = rng.standard_normal((rows, d0)).astype(np.float32)
    if dtype == "bf16":
        h = synth.f32_to_bf16_bits(h)
    u = rng.standard_normal((rows, n)).astype(np.float32)
    W = (rng.standard_normal((d1, n)) / np.sqrt(n)).astype(np.float32)
    got = extend(ebr, h, u, W)
    ref = oracle.ipnn_extend(h, u, W)
    g = synth.bf16_bits_to_f32(got).astype(np.float64) if dtype == "bf16" else got.astype(np.float64)
    assert (g[:, :d0] == ref[:, :d0]).all()                          # the tower part is copied
    bound = n * 2.0 ** -24 * (np.abs(u).astype(np.float64) @ np.abs(W).astype(np.float64).T)
    if dtype == "bf16":
        bound = bound + 2.0 ** -8 * np.abs(ref[:, d0:])              # one bf16 rounding
    assert (np.abs(g[:, d0:] - ref[:, d0:]) <= bound + 1e-30).all()


def test_query_with_ipnn_extended_towers(ebr):
    rng = np.random.default_rng(12)
    inv, users = synth.make_config("C3", mode="real", n_ads=200_000, batch=40)
    d0, n, d1 = inv.d, 24, 64                                        # h~ width 192
    v = rng.standard_normal((inv.n_ads, n)).astype(np.float32)
    uu = rng.standard_normal((users.batch, n)).astype(np.float32)
    Wv = (rng.standard_normal((d1, n)) / np.sqrt(n) / 4).astype(np.float32)
    Wu = (rng.standard_normal((d1, n)) / np.sqrt(n) / 4).astype(np.float32)
    ad_ext = extend(ebr, inv.ad_emb, v, Wv)
    user_ext = extend(ebr, users.user_emb, uu, Wu)
    inv2 = synth.Inventory(inv.n_ads, d0 + d1, inv.dtype, ad_ext, inv.ad_feat, inv.field_card, inv.cross_w,
                           inv.perm_seed)
    users2 = synth.Users(users.batch, users.slots, user_ext, users.user_feat, users.user_x)
    idx = ebr.Index.of(inv2)
    (ids, sc), _ = run(ebr, idx, users2, 500)
    check_many(oracle.Oracle.of(inv2), users2, ids, sc, 500, "real", sel=range(0, 40, 4))
