"""Ad-inventory sharding across the GPUs of one box (not in the paper, whose
operator runs on one T4).

Each rank owns a contiguous, 128-aligned ad range, builds its own index (ids stay global through
ad_begin), scores its shard for the full user batch and emits its local top-K as packed keys
kappa = (ord(score) << 32) | (0xFFFFFFFF - global_id).  ONE collective per batch -- an all-gather
of B*K 64-bit keys per rank (NCCL over NVLink/NVSwitch) -- then the merge kernel selects the
global top-K of the G*K keys per user.  kappa is unique per ad, so the merged answer equals the
single-GPU answer bit for bit.  The host logic here is plumbing only: every score, key and merge
is computed by the CUDA library.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

ALIGN = 128


def shard_range(n_ads: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's ads: ceil(N / G) rounded up to a multiple of 128 per rank."""
    per = ((n_ads + world - 1) // world + ALIGN - 1) // ALIGN * ALIGN
    lo = min(n_ads, rank * per)
    hi = min(n_ads, (rank + 1) * per)
    return lo, hi


def gather_keys(local_keys: torch.Tensor, group=None) -> torch.Tensor:
    """[B][K] int64 (kappa bits) per rank -> [G][B][K] on every rank."""
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(local_keys.shape), dtype=local_keys.dtype, device=local_keys.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local_keys.contiguous(), group=group)
    else:                                   # gloo (CPU tests): list form
        dist.all_gather(list(out.unbind(0)), local_keys.contiguous(), group=group)
    return out


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

    def workspace(self, batch: int, slots: int, k: int) -> torch.Tensor:
        key = (batch, slots, k)
        if key not in self._ws:
            self._ws[key] = self._ebr.new_workspace(self.index, batch, slots, k, device=self.device)
        return self._ws[key]

    def query(self, user_emb, user_feat, user_x, k: int, out_ids, out_scores, stream=None,
              local_keys=None, gathered=None):
        ebr = self._ebr
        B, F, S = user_feat.shape
        ws = self.workspace(B, S, k)
        if self.world == 1:
            ebr.score_topk(self.index, user_emb, user_feat, user_x, k, out_ids, out_scores, ws, stream)
            return
        if local_keys is None:
            local_keys = torch.empty((B, k), dtype=torch.int64, device=self.device)
        ebr.score_topk_keys(self.index, user_emb, user_feat, user_x, k, local_keys, ws, stream)
        if gathered is None:
            gathered = torch.empty((self.world, B, k), dtype=torch.int64, device=self.device)
        ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.current_stream())
        with ctx:
            if dist.get_backend(self.group) == "nccl":
                dist.all_gather_into_tensor(gathered, local_keys, group=self.group)
            else:
                dist.all_gather(list(gathered.unbind(0)), local_keys, group=self.group)
        ebr.merge_topk(gathered, self.world, B, k, out_ids, out_scores, stream)
