"""Ad-inventory sharding across the GPUs of one box (not in the paper, whose
operator runs on one T4).

Each rank owns a contiguous, 128-aligned ad range, builds its own index (ids stay global through
ad_begin), scores its shard for the full user batch and emits its local top-K as packed keys
kappa = (ord(score) << 32) | (0xFFFFFFFF - global_id).  One exchange per batch, then the merge
kernel selects the global top-K per user.  kappa is unique per ad, so the merged answer equals the
single-GPU answer bit for bit.  Two exchanges:

  full       one all-gather of B*K keys per rank (NCCL over NVLink/NVSwitch) + ebr_merge_topk;
  threshold  for large B*K: all-gather each rank's ceil(K/G)-th key per user (8*B bytes), the
             library packs only the local keys >= theta_u = min over ranks (a lower bound of the
             global K-th key, reading R24), all-gather of the counts and of the packed lists
             (padded to the largest rank total: one small all_reduce, a host sync), then
             ebr_merge_topk_packed -- ~8*B*K*(1+eps) bytes received instead of 8*G*B*K.

With overlap=True the exchange and the merge run on a side stream, so the next batch's scoring
on the caller's stream overlaps them (double-buffered key buffers); the returned event marks the
outputs final.  The host logic here is plumbing only: every score, key, threshold, pack and merge
is computed by the CUDA library.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

ALIGN = 128
THRESHOLD_BYTES = 64 << 20      # "auto": threshold exchange once a full gather would exceed this


def shard_range(n_ads: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's ads: ceil(N / G) rounded up to a multiple of 128 per rank."""
    per = ((n_ads + world - 1) // world + ALIGN - 1) // ALIGN * ALIGN
    lo = min(n_ads, rank * per)
    hi = min(n_ads, (rank + 1) * per)
    return lo, hi


def _all_gather(out: torch.Tensor, t: torch.Tensor, group=None):
    """out[G, ...] <- t from every rank.  NCCL: in place on the device; gloo (CPU tests and the
    one-GPU multi-process tests): through host copies."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return
    ht = t.detach().to("cpu").contiguous()
    parts = [torch.empty_like(ht) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, ht, group=group)
    out.copy_(torch.stack(parts).to(out.device))


def gather_keys(local_keys: torch.Tensor, group=None) -> torch.Tensor:
    """[B][K] int64 (kappa bits) per rank -> [G][B][K] on every rank."""
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(local_keys.shape), dtype=local_keys.dtype, device=local_keys.device)
    _all_gather(out, local_keys, group)
    return out


class _Buffers:
    def __init__(self, world, B, k, device):
        self.keys = torch.empty((B, k), dtype=torch.int64, device=device)
        self.gathered = torch.empty((world, B, k), dtype=torch.int64, device=device)
        self.kq = torch.empty((B,), dtype=torch.int64, device=device)
        self.kq_all = torch.empty((world, B), dtype=torch.int64, device=device)
        self.count = torch.empty((B,), dtype=torch.int32, device=device)
        self.off = torch.empty((B + 1,), dtype=torch.int32, device=device)
        self.packed = torch.empty((B * k,), dtype=torch.int64, device=device)
        self.count_all = torch.empty((world, B), dtype=torch.int32, device=device)
        self.free = None            # event: the side stream finished with this set


class ShardedIndex:
    """This rank's shard of a global inventory; query() returns the global top-K on every rank."""

    def __init__(self, inv, rank: int, world: int, device: int = 0, group=None):
        from . import ebr   # the CUDA library (raises if it is not built)
        self._ebr = ebr
        self.rank, self.world, self.group = rank, world, group
        self.lo, self.hi = shard_range(inv.n_ads, world, rank)
        if self.hi <= self.lo:
            raise ValueError("empty shard: more ranks than 128-ad blocks")
        self.index = ebr.Index.of(inv, lo=self.lo, hi=self.hi, device=device)
        self.device = torch.device("cuda", device)
        self._ws = {}
        self._bufs = {}
        self._flip = 0
        self.comm_stream = None

    def workspace(self, batch: int, slots: int, k: int) -> torch.Tensor:
        key = (batch, slots, k)
        if key not in self._ws:
            self._ws[key] = self._ebr.new_workspace(self.index, batch, slots, k, device=self.device)
        return self._ws[key]

    def _buffers(self, B, k, overlap):
        key = (B, k)
        if key not in self._bufs:
            self._bufs[key] = [_Buffers(self.world, B, k, self.device) for _ in range(2)]
        sets = self._bufs[key]
        if overlap:
            self._flip ^= 1
            return sets[self._flip]
        return sets[0]

    def exchange_mode(self, B: int, k: int, exchange: str = "auto") -> str:
        if exchange != "auto":
            return exchange
        return "threshold" if 8 * self.world * B * k > THRESHOLD_BYTES else "full"

    def query(self, user_emb, user_feat, user_x, k: int, out_ids, out_scores, stream=None,
              local_keys=None, gathered=None, exchange: str = "auto", overlap: bool = False):
        """Global top-k of every user into out_ids / out_scores (device, [B][k]).  Returns an event
        recorded once the outputs are final; without overlap `stream` already waits for it."""
        ebr = self._ebr
        B, F, S = user_feat.shape
        ws = self.workspace(B, S, k)
        stream = stream or torch.cuda.current_stream(self.device)
        if self.world == 1:
            ebr.score_topk(self.index, user_emb, user_feat, user_x, k, out_ids, out_scores, ws, stream)
            ev = torch.cuda.Event()
            ev.record(stream)
            return ev
        mode = self.exchange_mode(B, k, exchange)
        buf = self._buffers(B, k, overlap)
        keys = local_keys if local_keys is not None else buf.keys
        if buf.free is not None:
            stream.wait_event(buf.free)          # the side stream finished with this buffer set
        ebr.score_topk_keys(self.index, user_emb, user_feat, user_x, k, keys, ws, stream)
        if overlap:
            if self.comm_stream is None:
                self.comm_stream = torch.cuda.Stream(device=self.device)
            cs = self.comm_stream
            cs.wait_stream(stream)
        else:
            cs = stream
        with torch.cuda.stream(cs):
            if mode == "full":
                g = gathered if gathered is not None else buf.gathered
                _all_gather(g, keys, self.group)
                ebr.merge_topk(g, self.world, B, k, out_ids, out_scores, cs)
            else:
                G = self.world
                ebr.exchange_kth(keys, G, buf.kq, cs)
                _all_gather(buf.kq_all, buf.kq, self.group)
                ebr.exchange_pack(keys, buf.kq_all, G, buf.count, buf.off, buf.packed, cs)
                t_max = max(1, self._max_total(buf.off[B:B + 1].to(torch.int64)))
                send = buf.packed[:t_max]
                recv = torch.empty((G, t_max), dtype=torch.int64, device=self.device)
                _all_gather(recv, send, self.group)
                _all_gather(buf.count_all, buf.count, self.group)
                ebr.merge_topk_packed(recv, buf.count_all, G, B, k, out_ids, out_scores, cs)
            ev = torch.cuda.Event()
            ev.record(cs)
        buf.free = ev
        if not overlap:
            stream.wait_event(ev)
        return ev

    def _max_total(self, tot: torch.Tensor) -> int:
        """max over ranks of the packed totals (host-visible: sizes the padded all-gather)."""
        if dist.get_backend(self.group) == "nccl":
            t = tot.clone()
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            return int(t.item())
        t = tot.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return int(t.item())
