"""Per-kernel device times of one batched-path call (torch profiler-free: CUDA events around the
whole call + ncu gives the breakdown)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_22460_b200 import ebr, synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else None
n = int(sys.argv[3]) if len(sys.argv) > 3 else None
t = time.time()
inv, users = synth.make_config(cfg, batch=B, n_ads=n)
print("gen", time.time() - t, flush=True)
c = synth.CONFIGS[cfg]
t = time.time()
idx = ebr.Index.of(inv)
print("build", time.time() - t, idx.stats(), flush=True)
Bn, F, S = users.user_feat.shape
dev = torch.device("cuda")
emb = torch.from_numpy(users.user_emb.view(np.int16)).to(dev)
feat = torch.from_numpy(users.user_feat).to(dev)
x = torch.from_numpy(users.user_x).to(dev)
ws = ebr.new_workspace(idx, Bn, S, c.k)
ids = torch.empty((Bn, c.k), dtype=torch.int32, device=dev)
sc = torch.empty((Bn, c.k), dtype=torch.float32, device=dev)
for it in range(int(os.environ.get("ITERS", "5"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ebr.score_topk(idx, emb, feat, x, c.k, ids, sc, ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"call {it}: {ms:.3f} ms  -> {Bn / ms * 1e3:.0f} users/s", flush=True)
