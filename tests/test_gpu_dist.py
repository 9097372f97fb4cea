"""Multi-GPU data plane, end to end on ONE GPU: two ranks (processes) with a gloo process group,
each building its shard's index on cuda:0 and running dist.ShardedIndex.query (local top-K keys
through the C-ABI, the exchange, the merge kernel).  Checked element by element against the CPU
oracle (exact mode: bit-exact ids and scores, Eq. 9, top k l.157) for both
exchanges (full all-gather; threshold exchange, reading R24) and with the exchange overlapped on a
side stream.  The ranks' kernels never wait on each other (the collectives are host-side gloo)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2511_22460_b200 import synth  # noqa: E402
from tests.parity import check_many  # noqa: E402

CASES = [("C3", 200_000, 40, 300), ("C2", 60_000, 3, 500), ("C4", 150_000, 64, 1000)]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2511_22460_b200.dist import ShardedIndex
    dev = torch.device("cuda", 0)
    for ci, (cfg, n, b, k) in enumerate(CASES):
        inv, users = synth.make_config(cfg, mode="exact", n_ads=n, batch=b)
        sh = ShardedIndex(inv, rank, world, device=0)
        emb_np = users.user_emb
        emb = torch.from_numpy(emb_np.view(np.int16) if emb_np.dtype == np.uint16 else emb_np).to(dev)
        feat = torch.from_numpy(users.user_feat).to(dev)
        x = torch.from_numpy(users.user_x).to(dev)
        for mode in ("full", "threshold"):
            for overlap in (False, True):
                ids = torch.empty((b, k), dtype=torch.int32, device=dev)
                sc = torch.empty((b, k), dtype=torch.float32, device=dev)
                st = torch.cuda.Stream()
                ev = sh.query(emb, feat, x, k, ids, sc, st, exchange=mode, overlap=overlap)
                if overlap:          # a second batch in flight while the first one's exchange runs
                    ids2 = torch.empty_like(ids)
                    sc2 = torch.empty_like(sc)
                    ev2 = sh.query(emb, feat, x, k, ids2, sc2, st, exchange=mode, overlap=True)
                    ev2.synchronize()
                ev.synchronize()
                torch.cuda.synchronize()
                if rank == 0:
                    np.save(os.path.join(outdir, f"{ci}_{mode}_{int(overlap)}_ids.npy"), ids.cpu().numpy())
                    np.save(os.path.join(outdir, f"{ci}_{mode}_{int(overlap)}_sc.npy"), sc.cpu().numpy())
                    if overlap:
                        np.save(os.path.join(outdir, f"{ci}_{mode}_2_ids.npy"), ids2.cpu().numpy())
        sh.index.close()
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_one_gpu_equal_oracle(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    for ci, (cfg, n, b, k) in enumerate(CASES):
        inv, users = synth.make_config(cfg, mode="exact", n_ads=n, batch=b)
        o = oracle.Oracle.of(inv)
        ref = None
        for mode in ("full", "threshold"):
            for ov in (0, 1):
                ids = np.load(tmp_path / f"{ci}_{mode}_{ov}_ids.npy")
                sc = np.load(tmp_path / f"{ci}_{mode}_{ov}_sc.npy")
                if ref is None:
                    assert check_many(o, users, ids, sc, k, "exact") == 0
                    ref = (ids, sc)
                else:
                    assert (ids == ref[0]).all() and (sc == ref[1]).all(), (cfg, mode, ov)
                if ov:
                    assert (np.load(tmp_path / f"{ci}_{mode}_2_ids.npy") == ref[0]).all()
