"""World-size-2 CPU test (gloo) of the multi-GPU plumbing: shard ranges, the key all-gather and the
A7 invariant "merge of the shard top-Ks == the top-K of the union" -- with the oracle standing in
for the per-shard GPU scorer (test infrastructure) and a numpy merge as the reference."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2511_22460_b200 import synth
from paper_2511_22460_b200.dist import gather_keys, shard_range


def _kappa(scores_fp32: np.ndarray, gids: np.ndarray) -> np.ndarray:
    """Reference packing of (score, id) per the ABI (include/ebr.h): ord(s) << 32 | ~id."""
    u = scores_fp32.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = np.where(u == 0x80000000, 0, u)
    neg = (u & 0x80000000) != 0
    o = np.where(neg, (~u) & 0xFFFFFFFF, u | 0x80000000)
    return (o << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - gids.astype(np.uint64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, k, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inv, users = synth.make_config("C1", mode="exact", n_ads=3_001, batch=3)
    lo, hi = shard_range(inv.n_ads, world, rank)
    o = oracle.Oracle(inv.ad_emb[lo:hi], inv.ad_feat[lo:hi], inv.field_card, inv.cross_w, id_base=lo)
    ids, r, _ = o.topk(users.user_emb, users.user_feat, users.user_x, k)
    keys = np.where(ids >= 0, _kappa(r.astype(np.float32), np.maximum(ids, 0)), 0).astype(np.uint64)
    g = gather_keys(torch.from_numpy(keys.view(np.int64)))
    if rank == 0:
        result.put(g.numpy().view(np.uint64))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_shard_gather_merge(world):
    k = 120
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert gathered.shape == (world, 3, k)
    # reference merge: top-K of the union of the shard lists (keys are unique; 0 = padding)
    inv, users = synth.make_config("C1", mode="exact", n_ads=3_001, batch=3)
    o = oracle.Oracle.of(inv)
    ids, r, _ = o.topk(users.user_emb, users.user_feat, users.user_x, k)
    for b in range(3):
        union = np.sort(gathered[:, b, :].ravel())[::-1][:k]
        ref = _kappa(r[b].astype(np.float32), ids[b])
        assert (union == ref).all()


def test_shard_ranges_cover_and_align():
    for n in (1, 127, 128, 129, 10_000, 1_000_003):
        for g in (1, 2, 3, 8):
            rs = [shard_range(n, g, r) for r in range(g)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (a, b), (c, d) in zip(rs, rs[1:]):
                assert b == c
            for a, b in rs[:-1]:
                assert a % 128 == 0 and (b - a) % 128 == 0 or b == n
