"""Phase breakdown of the latency-path kernel (EBR_PHASE_TIMERS=1: per-CTA globaltimer stamps).

Prints, per phase stamp, the min / median / max over CTAs of (stamp - earliest CTA start), in us.
"""
import os
import sys

os.environ["EBR_PHASE_TIMERS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import warnings
warnings.simplefilter('ignore')
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

# replica of small_layout() (ebr_small.cu), kSmallMaxB = 4, kHistBins = 2048
st = idx.stats()
sms = torch.cuda.get_device_properties(0).multi_processor_count
n_pad = (st["n_ads"] + 127) // 128 * 128
al = lambda v: (v + 255) & ~255
o = al(16 + 16 * 8)
off_hist = o; o = al(o + 4 * 2048 * 4)
off_count = o; o = al(o + 4 * (sms + 1) * 4)
o = al(o + 4 * n_pad * 4)
o = al(o + 4 * n_pad * 8)
off_timers = o
R = (st["n_ads"] + sms - 1) // sms
R = max(32, (R + 31) & ~31)
n_ranges = (st["n_ads"] + R - 1) // R

names = {0: "start", 1: "plan", 2: "wide_sample", 15: "sample_pub", 3: "deep_done", 4: "stream_end",
         7: "sample_wait", 14: "thresh_done", 8: "compact_done", 11: "last:seg_scan",
         12: "last:staged", 13: "last:selected", 10: "last:end"}
acc = []
for it in range(30):
    if not os.environ.get("NOFLUSH"):
        flush.sum()
    torch.cuda.synchronize()
    ebr.score_topk(idx, emb, feat, x, c.k, ids, sc, ws)
    torch.cuda.synchronize()
    t = ws[off_timers:off_timers + n_ranges * 16 * 8].cpu().numpy().view(np.uint64).reshape(n_ranges, 16)
    t = t.astype(np.float64)
    t0 = t[:, 0].min()
    v = (t - t0) / 1e3
    v[t == 0] = np.nan                        # stamp not reached by that CTA (e.g. only the last CTA selects)
    acc.append(np.stack([np.nanmin(v, 0), np.nanmedian(v, 0), np.nanmax(v, 0)], 1))   # [16][3]
a = np.nanmedian(np.array(acc[5:]), axis=0)   # [16][3], median over calls
cc = ws[off_count:off_count + 4 * n_ranges].cpu().numpy().view(np.uint32)
print("candidates user 0:", int(cc.sum()), "max per CTA", int(cc.max()))
print(f"{'stamp':14s} {'min':>8s} {'median':>8s} {'max':>8s}  (us since first CTA start; median over calls)")
for i in range(16):
    if i not in names:
        names[i] = f"stamp{i}"
for i in [0, 1, 2, 15, 3, 4, 6, 7, 5, 14, 8, 9, 11, 12, 13, 10]:
    print(f"{names[i]:14s} {a[i, 0]:8.2f} {a[i, 1]:8.2f} {a[i, 2]:8.2f}")
print("stats", st)
