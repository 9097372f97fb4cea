"""Phase breakdown of the latency-path kernel (EBR_PHASE_TIMERS=1 globaltimer stamps)."""
import os
import sys

os.environ["EBR_PHASE_TIMERS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_22460_b200 import ebr, synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
B = int(sys.argv[2]) if len(sys.argv) > 2 else None
inv, users = synth.make_config(cfg, batch=B)
c = synth.CONFIGS[cfg]
idx = ebr.Index.of(inv)
Bn, F, S = users.user_feat.shape
dev = torch.device("cuda")
emb = torch.from_numpy(users.user_emb.view(np.int16) if users.user_emb.dtype == np.uint16 else users.user_emb).to(dev)
feat = torch.from_numpy(users.user_feat).to(dev)
x = torch.from_numpy(users.user_x).to(dev)
ws = ebr.new_workspace(idx, Bn, S, c.k)
ids = torch.empty((Bn, c.k), dtype=torch.int32, device=dev)
sc = torch.empty((Bn, c.k), dtype=torch.float32, device=dev)
flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)   # 256 MiB, read to flush L2 clean
names = ["start", "plan", "wide_done", "deep_done", "B_end", "sync1", "fuse_end", "sync2", "compact_end", "sync3", "select_end", "sel_staged", "sel_radix", "sel_sorted", "thresh_done"]
acc = []
for it in range(30):
    if not os.environ.get("NOFLUSH"):
        flush.sum()
    torch.cuda.synchronize()
    ebr.score_topk(idx, emb, feat, x, c.k, ids, sc, ws)
    torch.cuda.synchronize()
    t = ws[16:16 + 15 * 8].cpu().numpy().view(np.uint64).astype(np.float64)
    acc.append((t - t[0]) / 1e3)
a = np.median(np.array(acc[5:]), axis=0)
cc = ws[65792:65792 + 4 * 149].cpu().numpy().view(np.uint32)
print("candidates user 0:", int(cc[:148].sum()), "max per CTA", int(cc[:148].max()))
for n, v in zip(names, a):
    print(f"{n:12s} {v:8.2f} us")
print("stats", idx.stats())
