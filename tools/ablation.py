"""NEXT-3 ablation on B200: the paper's inverted list (Alg. 1-2) vs this library's chunk codec,
the same HitMatch algorithm (flat work space, fp32 AtomicAdd into a global score array) for one
user at a time -- the shape of the paper's Table 2 (QPS and latency of the HitMatch
operator, preprocessing time).  Prints one JSON line per config."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_22460_b200 import ebr, synth
from tests.test_gpu_paper import items_of

dev = torch.device("cuda")
for cfg in sys.argv[1:] or ["C2"]:
    inv, users = synth.make_config(cfg, mode="real", batch=64)
    t = time.perf_counter(); idx = ebr.Index.of(inv); t_chunk = time.perf_counter() - t
    t = time.perf_counter(); pidx = ebr.PaperIndex(inv.ad_feat, inv.field_card); t_paper = time.perf_counter() - t
    qs = [items_of(inv, users.user_feat[b], users.user_x[b]) for b in range(users.batch)]
    qk = [torch.from_numpy(k).to(dev) for k, _ in qs]
    qw = [torch.from_numpy(w).to(dev) for _, w in qs]
    out = torch.empty(inv.n_ads, dtype=torch.float32, device=dev)
    res = {}
    for name, fn in (("paper", lambda i: ebr.paper_hitmatch(pidx, qk[i], qw[i], out)),
                     ("chunk", lambda i: ebr.chunk_hitmatch(idx, qk[i], qw[i], out))):
        for i in range(8):
            fn(i)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(256)]
        for j, (a, b) in enumerate(ev):
            a.record(); fn(j % len(qs)); b.record()
        torch.cuda.synchronize()
        ms = np.array([a.elapsed_time(b) for a, b in ev])
        res[name] = {"us_mean": float(ms.mean() * 1e3), "us_p50": float(np.median(ms) * 1e3),
                     "qps": float(1e3 / ms.mean())}
    st = idx.stats()
    info = pidx.info()
    print(json.dumps({"config": cfg, "n_ads": inv.n_ads, "nnz": st["nnz"], "items_per_query": float(np.mean([len(k) for k, _ in qs])),
                      "paper": dict(res["paper"], index_bytes=info["bytes"], build_ms_host=t_paper * 1e3,
                                    blocks_per_group=info["blocks_per_group"]),
                      "chunk": dict(res["chunk"], index_bytes=st["index_bytes"], build_ms_host=t_chunk * 1e3,
                                    chunks=st["chunks"]),
                      "timing": "CUDA events around each call (memset of the score array + kernel), 256 calls, one user each"}),
          flush=True)
