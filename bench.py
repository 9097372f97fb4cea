#!/usr/bin/env python
"""Benchmark of the Wide & Deep retrieval hot path (arXiv 2511.22460) on B200.

One step = one batch of users scored against the whole inventory (wide through the compressed
inverted list + deep dual-tower inner product + fused top-K), i.e. every SURVEY.md §8(a) row;
for N > 1 GPUs the inventory is sharded by ad range (strong scaling of a fixed inventory) and
each step adds the NCCL all-gather of the per-shard top-K keys and the merge kernel.

Default workload: BASELINE.json config 2 ("1M ads, d=64, 32 cross features, batch 1, K=500 on
1 B200 (latency path)").  Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2511_22460_b200 import synth  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--mode", default="real")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="few steps, no side measurements (for ncu)")
    ap.add_argument("--graph", action="store_true",
                    help="replay a CUDA graph of the library call each step (latency path, 1 GPU); measured "
                         "no faster than the direct call (profiles/r01_mb_launch.txt), so off by default")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5:   # first sample before timing starts
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def algorithmic_bytes(ebr, inv, users, idx_stats, lo, hi):
    """N_s*d*e (embeddings, once) + P_U (encoded postings of the batch's
    distinct keys in the shard: 8-byte chunk headers + payload words) + inputs + outputs."""
    kco, kwo, hdr, pay = ebr.encode_host(inv.ad_feat[lo:hi], inv.field_card)
    base = np.concatenate([[0], np.cumsum(inv.field_card)[:-1]]).astype(np.int64)
    F, S = users.user_feat.shape[1:]
    keys = set()
    for b in range(users.batch):
        for f in range(F):
            for s in range(S):
                v = users.user_feat[b, f, s]
                if v >= 0:
                    keys.add(int(base[f] + v))
    keys = np.array(sorted(keys), np.int64)
    nch = (kco[keys + 1].astype(np.int64) - kco[keys]).sum()
    # payload words of a key = next key's word base - this one's (keys are laid out in order)
    wend = np.append(kwo.astype(np.int64), len(pay))
    words = (wend[keys + 1] - wend[keys]).sum()
    hits = 0
    esz = 2 if inv.dtype == "bf16" else 4
    emb = (hi - lo) * idx_stats["d_pad"] * esz
    postings = int(nch) * 8 + int(words) * 4 + len(keys) * 12
    io = users.batch * (inv.d * esz + 8 * F * S)
    return emb, postings, io


def run_reference(args, cfg, rank, world):
    """Reference arm: the CPU oracle as it stands, on this host's cores (no GPU).  Each step is a
    bounded sample of the workload -- min(B, cores) users of the batch scored against a seeded
    prefix of the inventory sized so the whole run takes ~2 minutes -- and users/s is rescaled to
    the full inventory by ads-scored/s (the oracle's cost is linear in N plus an N log N sort)."""
    if rank != 0:
        return
    import oracle
    B = args.batch or cfg.batch
    K = args.k or cfg.k
    inv, users = synth.make_config(cfg, mode=args.mode, batch=B)
    threads = os.cpu_count() or 1
    nu = max(1, min(B, threads))
    o_full = oracle.Oracle.of(inv)
    t = time.perf_counter()
    o_full.topk(users.user_emb[:1], users.user_feat[:1], users.user_x[:1], K, threads=1)
    per_user_full = time.perf_counter() - t
    budget = max(0.02, 120.0 / max(args.steps + args.warmup, 1))
    n_sub = int(min(inv.n_ads, max(K, inv.n_ads * budget / max(per_user_full, 1e-6))))
    o = oracle.Oracle(inv.ad_emb[:n_sub], inv.ad_feat[:n_sub], inv.field_card, inv.cross_w)
    for s in range(args.warmup):
        o.topk(users.user_emb[:1], users.user_feat[:1], users.user_x[:1], K, threads=1)
    times = []
    for s in range(args.steps):
        sel = [(s * nu + j) % B for j in range(nu)]
        t = time.perf_counter()
        o.topk(users.user_emb[sel], users.user_feat[sel], users.user_x[sel], K, threads=nu)
        times.append(time.perf_counter() - t)
    tot = sum(times)
    ads_s = nu * n_sub * args.steps / tot
    users_s = ads_s / inv.n_ads
    line = {
        "impl": "reference",
        "metric": "users_per_s", "value": users_s, "unit": "users/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * B / users_s,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": f"synthetic ({args.mode} mode, seeded generator)",
        "config": config_dict(cfg, B, K, world),
        "ads_scored_per_s": ads_s,
        "cpu_baseline": {"value": users_s, "unit": "users/s", "cores": nu, "kind": "oracle",
                         "sample": f"per step {nu} user(s) x the first {n_sub} of {inv.n_ads} ads "
                                   f"(rescaled by ads-scored/s); full-inventory single-thread "
                                   f"{per_user_full:.3f} s/user"},
        "e2e": {"value": users_s, "unit": "users/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def config_dict(cfg, B, K, world):
    return {"workload": f"{cfg.name}: {cfg.n_ads} ads, d={cfg.d} {cfg.dtype}, {cfg.n_fields} cross "
                        f"features (Zipf alpha={cfg.alpha}), batch {B}, K={K}",
            "n_ads": cfg.n_ads, "d": cfg.d, "emb_dtype": cfg.dtype, "cross_features": cfg.n_fields,
            "slots_per_field": cfg.slots, "zipf_alpha": cfg.alpha, "batch": B, "k": K,
            "parallelism": f"ad-shard x{world}",
            "l2": "flushed between steps by reading a 256 MiB buffer (clean lines, no write-back), "
                  "outside the per-step events; A itself is larger than L2"}


def cpu_baseline(cfg, inv, users, K, budget_s=15.0):
    import oracle
    o = oracle.Oracle.of(inv)
    threads = os.cpu_count() or 1
    t = time.perf_counter()
    o.topk(users.user_emb[:1], users.user_feat[:1], users.user_x[:1], K, threads=1)
    one = time.perf_counter() - t
    n = int(max(1, min(threads * 4, budget_s / max(one, 1e-3) * threads / 1.5)))
    rng = np.random.default_rng(0)
    B = users.batch
    sel = rng.integers(0, B, n) if B > 1 else np.zeros(n, np.int64)
    t = time.perf_counter()
    o.topk(users.user_emb[sel], users.user_feat[sel], users.user_x[sel], K, threads=min(threads, n))
    dt = time.perf_counter() - t
    return {"value": n / dt, "unit": "users/s", "cores": min(threads, n), "kind": "oracle",
            "sample": f"{n} users (drawn from the batch) x all {inv.n_ads} ads, brute-force sort",
            "single_thread_s_per_user": one}


def main():
    args = parse()
    cfg = synth.CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    import torch
    import torch.distributed as dist
    from paper_2511_22460_b200 import ebr

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    B = args.batch or cfg.batch
    K = args.k or cfg.k
    inv, users = synth.make_config(cfg, mode=args.mode, batch=B)
    N = inv.n_ads
    from paper_2511_22460_b200.dist import ShardedIndex
    shard = ShardedIndex(inv, rank, world, device=local)
    idx = shard.index
    lo, hi = shard.lo, shard.hi
    st = idx.stats()
    stream = torch.cuda.Stream(device=dev)
    emb_np = users.user_emb
    emb = torch.from_numpy(emb_np.view(np.int16) if emb_np.dtype == np.uint16 else emb_np).to(dev)
    feat = torch.from_numpy(users.user_feat).to(dev)
    x = torch.from_numpy(users.user_x).to(dev)
    S = users.slots
    ws = shard.workspace(B, S, K)
    ids = torch.empty((B, K), dtype=torch.int32, device=dev)
    sc = torch.empty((B, K), dtype=torch.float32, device=dev)
    keys = torch.empty((B, K), dtype=torch.int64, device=dev)
    gathered = torch.empty((world, B, K), dtype=torch.int64, device=dev)
    flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)   # 256 MiB, READ between steps
    flush_out = torch.empty((), dtype=torch.float32, device=dev)

    def call():
        shard.query(emb, feat, x, K, ids, sc, stream, local_keys=keys, gathered=gathered)

    step = call
    # --graph (1 GPU, latency path): replay a CUDA graph of the library call (the same cooperative
    # kernel, enqueued without the per-call host work).  The batched path synchronises once per
    # call (overflow check) and is always launched directly.
    use_graph = (world == 1 and args.graph
                 and idx.query_launches(B, S, K) == (B + 3) // 4)
    for _ in range(max(args.warmup, 3)):
        call()
    torch.cuda.synchronize()
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            call()
        torch.cuda.synchronize()

        def step():
            with torch.cuda.stream(stream):
                graph.replay()
        for _ in range(3):
            step()
        torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    hbm_peak, peak_kind = peaks()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        t0 = time.perf_counter()
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                torch.sum(flush, dim=0, out=flush_out)           # evict L2 clean (outside the events)
                ev[i][0].record(stream)
            step()
            with torch.cuda.stream(stream):
                ev[i][1].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if world > 1:
        dist.barrier()
    per = np.array([a.elapsed_time(b) for a, b in ev])        # ms, device side
    tot_ms = float(per.sum())
    t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms = float(t.item())
    ms_step = tot_ms / args.steps
    users_s = B * args.steps / (tot_ms / 1e3)

    line = None
    batched = idx.query_launches(B, S, K) != (B + 3) // 4
    kernel_label = ("whole batched step per 128-user group: plan, span, wide_smem, gemm_kernel<0> (sample), "
                    "theta, gemm_kernel<1> (tcgen05 + fused filter), final -- timed as one" if batched else
                    "small_kernel (fused plan+decode+wide+GEMV+fuse+top-K, 1 launch per <=4 users)")
    if rank == 0:
        emb_b, post_b, io_b = algorithmic_bytes(ebr, inv, users, st, lo, hi)
        alg = emb_b + post_b + io_b + 8 * B * K
        achieved = alg / (ms_step / 1e3) / 1e9   # GB/s (per GPU: shard bytes / step time)
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                tr = json.load(f).get(cfg.name)
            if tr and tr.get("world", 1) == world and tr.get("batch") == B:
                traffic = tr["dram_bytes_per_launch"]
        except Exception:
            pass
        line = {
            "metric": "users_per_s", "value": users_s, "unit": "users/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if cfg.dtype == "f32" else "bf16",
            "data": f"synthetic ({args.mode} mode, seeded Zipf generator of DESIGN.md)",
            "config": config_dict(cfg, B, K, world),
            "ads_scored_per_s": users_s * N,
            "latency_us": {"p50": float(np.percentile(per, 50) * 1e3),
                           "p99": float(np.percentile(per, 99) * 1e3),
                           "min": float(per.min() * 1e3)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic,
                         "peak_kind": peak_kind,
                         "kernel": kernel_label,
                         "alg_bytes_per_launch": alg,
                         "alg_bytes_split": {"embeddings": emb_b, "postings": post_b, "io": io_b + 8 * B * K}},
            "index": {"build_ms": st["build_ms"], "index_bytes": st["index_bytes"],
                      "nnz": st["nnz"], "chunks": st["chunks"]},
            "clocks": clk.summary(),
            "gpu_launches": args.steps * (idx.query_launches(B, S, K) + (1 if world > 1 else 0)),
            "launch": "cuda_graph replay of the C-ABI call" if use_graph else "direct C-ABI call per step",
            "wall_s_timed_region": wall,
        }
    # e2e through the public API with HOST buffers: N=1 -> the C-ABI host call (H2D, query, D2H,
    # sync inside the library); N>1 -> pinned H2D + sharded query (+ all-gather + merge) + D2H
    if not args.profile:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        h_emb = pin(emb_np.view(np.int16) if emb_np.dtype == np.uint16 else emb_np)
        h_feat, h_x = pin(users.user_feat), pin(users.user_x)
        h_ids = torch.empty((B, K), dtype=torch.int32).pin_memory()
        h_sc = torch.empty((B, K), dtype=torch.float32).pin_memory()
        if world == 1:
            wsh = ebr.new_workspace(idx, B, S, K, host=True)
            n_h = [h_emb.numpy(), h_feat.numpy(), h_x.numpy(), h_ids.numpy(), h_sc.numpy()]
            run_e2e = lambda: ebr.score_topk_host(idx, n_h[0], n_h[1], n_h[2], K, n_h[3], n_h[4], wsh, stream)  # noqa: E731
            timing = "host wall clock around ebr_score_topk_host (H2D + query + D2H + sync)"
        else:
            def run_e2e():
                with torch.cuda.stream(stream):
                    emb.copy_(h_emb, non_blocking=True)
                    feat.copy_(h_feat, non_blocking=True)
                    x.copy_(h_x, non_blocking=True)
                step()
                with torch.cuda.stream(stream):
                    h_ids.copy_(ids, non_blocking=True)
                    h_sc.copy_(sc, non_blocking=True)
                stream.synchronize()
            timing = "host wall clock: pinned H2D + sharded query + all-gather + merge + D2H + sync"
        for _ in range(3):
            run_e2e()
        e_ms = []
        n_e2e = min(args.steps, 500)
        for i in range(n_e2e):
            with torch.cuda.stream(stream):
                torch.sum(flush, dim=0, out=flush_out)
            stream.synchronize()
            if world > 1:
                dist.barrier()
            t = time.perf_counter()
            run_e2e()
            e_ms.append((time.perf_counter() - t) * 1e3)
        e_arr = torch.tensor([float(np.mean(e_ms))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_arr, op=dist.ReduceOp.MAX)
        if line is not None:
            line["e2e"] = {"value": B / (float(e_arr.item()) / 1e3), "unit": "users/s",
                           "h2d_bytes_per_step": int(h_emb.nbytes + h_feat.nbytes + h_x.nbytes),
                           "d2h_bytes_per_step": int(h_ids.nbytes + h_sc.nbytes),
                           "p50_us": float(np.percentile(e_ms, 50) * 1e3), "timing": timing}
    if rank == 0 and not args.no_cpu_baseline and not args.profile:
        line["cpu_baseline"] = cpu_baseline(cfg, inv, users, K)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
