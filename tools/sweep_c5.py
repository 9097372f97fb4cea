"""C5 sweep (BASELINE.json config 5): top-K K=10..10000 x user batch 1..1024 on 20M ads, one GPU.
Prints one JSON line per point (device-timed CUDA events, L2 flushed by a read between steps) with
the nvidia-smi clocks sampled while the point ran (bench.py's Clocks)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2511_22460_b200 import ebr, synth
from bench import Clocks

Bs = [int(x) for x in os.environ.get("BS", "1,4,16,64,256,1024").split(",")]
Ks = [int(x) for x in os.environ.get("KS", "10,100,1000,10000").split(",")]
steps = int(os.environ.get("STEPS", "5"))
t = time.time()
inv, users = synth.make_config("C5", batch=max(Bs))
print(json.dumps({"gen_s": time.time() - t}), flush=True)
t = time.time()
idx = ebr.Index.of(inv, device_build=os.environ.get("DEVICE_BUILD", "1") == "1")
print(json.dumps({"build_s": time.time() - t, "stats": idx.stats()}), flush=True)
dev = torch.device("cuda")
flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)
fo = torch.empty((), dtype=torch.float32, device=dev)
for B in Bs:
    emb = torch.from_numpy(users.user_emb[:B].view(np.int16)).to(dev)
    feat = torch.from_numpy(users.user_feat[:B]).to(dev)
    x = torch.from_numpy(users.user_x[:B]).to(dev)
    for K in Ks:
        ws = ebr.new_workspace(idx, B, users.slots, K)
        ids = torch.empty((B, K), dtype=torch.int32, device=dev)
        sc = torch.empty((B, K), dtype=torch.float32, device=dev)
        ebr.score_topk(idx, emb, feat, x, K, ids, sc, ws)
        torch.cuda.synchronize()
        ms = []
        with Clocks(0) as clk:
            for _ in range(steps):
                torch.sum(flush, dim=0, out=fo)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); ebr.score_topk(idx, emb, feat, x, K, ids, sc, ws); e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
        m = float(np.median(ms))
        batched = idx.query_launches(B, users.slots, K) != (B + 3) // 4
        print(json.dumps({"B": B, "K": K, "ms": m, "users_per_s": B / m * 1e3,
                          "ads_scored_per_s": B * inv.n_ads / m * 1e3,
                          "path": "tensor-core batched" if batched else "latency",
                          "clocks": clk.summary()}), flush=True)
        del ws
