"""Benchmark of the Multipole Attention decode path on B200 (BASELINE.json metric:
"decode attention us/step & speedup vs dense at 32K ctx; HBM GB/s vs peak").

Workload (configs[1]): Qwen3-8B attention shape -- 32 q-heads, 8 kv-heads (GQA x4), head_dim 128,
32K context, 1-level clustering (r = 16 -> ~2040 centroids / head), token budget B = 512,
rope theta 1e6, bf16 KV cache, batch 16 sequences per GPU.  Synthetic N(0,1) Q/K/V (random-init
model shape, torch seed 0 + rank).  The ledger is built by the GPU clustering path.

A step = one decode step of one attention layer for the whole batch: q rotation, centroid
lookup + budgeted selection, fused sparse-exact + centroid-replacement attention with the
split-KV merge, and the KV append of the step's token.  L2 is flushed (256 MB write, then a
256 MB read so no dirty flush lines are left to write back) before every timed step; each
step is timed with CUDA events on the engine stream.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

N > 1 (torchrun): every rank runs its own batch (replicas, batch-sharded: no collective on
the data path), barrier + max over ranks; `--workload c5` at N > 1 shards one long context
over the ranks instead.  `--impl reference` times the reference package itself (pure Python,
installed into baseline/_ref by __graft_entry__.build()) on rank 0's host cores, falling back to
the oracle port when it is not importable.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CALIB_STEPS = 0
METRIC = "decode attention µs/step & speedup vs dense at 32K ctx; HBM GB/s vs peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"],
                    help="BASELINE configs: c2 (default, the metric's config), c3 (R1-14B 64K 2-level), "
                         "c4 (online updates while generating), c5 (128K sequence-sharded over the ranks)")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--ctx", type=int, default=None)
    ap.add_argument("--budget", type=int, default=512)
    ap.add_argument("--page-size", type=int, default=None,
                    help="serve K_rot / V from a paged pool with this many tokens per page (shuffled pages)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline leg")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no CPU leg, no clocks)")
    a = ap.parse_args()
    dflt = {"c2": (16, 32768), "c3": (16, 65536), "c4": (8, 16384), "c5": (16, 131072)}[a.workload]
    a.batch = a.batch or dflt[0]
    a.ctx = a.ctx or dflt[1]
    if a.workload == "c4" and a.steps == 20:
        a.steps = 512  # spans four online-update events (L = 128)
    if a.workload == "c4":
        # warm-up covers one online-update event, so the timed steps see steady-state events (the
        # first event in a process also pays one-time lazy CUDA module loads and allocator growth)
        a.warmup = max(a.warmup, 130)
    return a


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload_cfg(args):
    from paper_2506_13059_b200.core import EngineConfig, HeadLayout, HierarchyConfig

    if getattr(args, "workload", "c2") == "c3":  # DeepSeek-R1-Distill-Qwen-14B attention: 40 q / 8 kv
        lay = HeadLayout(40, 8, 128)
        cfg = EngineConfig(token_budget=args.budget, rope_theta=1e6, seed=0,
                           hierarchy=HierarchyConfig(64, 8, 0.25))
        return lay, cfg
    lay = HeadLayout(32, 8, 128)
    cfg = EngineConfig(token_budget=args.budget, tokens_per_centroid=16, rope_theta=1e6, seed=0)
    return lay, cfg


def workload_label(args, world=1):
    b, ctx, B = args.batch, args.ctx, args.budget
    w = getattr(args, "workload", "c2")
    if w == "c3":
        return (f"C3: DeepSeek-R1-Distill-Qwen-14B attention shape 40q/8kv/d128, {ctx // 1024}K ctx, 2-level "
                f"r1=64/r2=8/p=0.25, B={B}, bf16, batch {b}/GPU")
    if w == "c4":
        return (f"C4: Qwen3-8B attention shape 32q/8kv/d128, {ctx // 1024}K prompt + generated tokens with online "
                f"cluster updates every L=128 steps, r=16, B={B}, bf16, batch {b}/GPU")
    if w == "c5":
        return (f"C5: Qwen3-8B attention shape 32q/8kv/d128, {ctx // 1024}K ctx KV-sequence-sharded over {world} "
                f"GPU(s) (NCCL all-gather merge), r=16, B={B}, bf16, batch {b}")
    return f"C2: Qwen3-8B attention shape 32q/8kv/d128, {ctx // 1024}K ctx, 1-level r=16, B={B}, bf16, batch {b}/GPU"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        if os.environ.get("BENCH_NO_SMI") == "1":  # experiments: no sampler
            return self
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        loaded = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------- CPU oracle leg


def cpu_oracle_time(lay, cfg, keys, values, queries, ledger_o, cache_len, n_steps=3):
    """Seconds per decode step of ONE ledger (1 sequence x 1 kv-head, its G q-heads) and of one
    dense-oracle step of the same ledger, timed with the numpy oracle on the host cores."""
    from oracle import mpa_oracle as O
    from paper_2506_13059_b200.core import HeadLayout

    one = HeadLayout(lay.group_size, 1, lay.head_dim)
    t0 = time.perf_counter()
    for t in range(n_steps):
        O.decode_step(queries[t], [ledger_o], [keys], [values], cache_len, t, cfg, one)
    sparse = (time.perf_counter() - t0) / n_steps
    t0 = time.perf_counter()
    pos = np.arange(cache_len)
    for g in range(lay.group_size):
        O.dense_attention(queries[0][g], cache_len, keys[:cache_len], values[:cache_len], pos, lay.head_dim,
                          cfg.rope_theta)
    dense = time.perf_counter() - t0
    return sparse, dense


def _import_reference():
    """The unmodified reference package, pip-installed into baseline/_ref (pure Python + numpy)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import multipole_attn  # noqa: F401

    return multipole_attn


def reference_arm(args, rank, world):
    """--impl reference: the REAL reference package (baseline/_ref, its own stock code path) on the
    host cores of rank 0: one kv-head ledger of the bench workload is built with
    clustering.build_prefill_index_head and decode steps run through
    attention.decode_step_attention; the per-ledger time is scaled to the batch (the reference
    loops kv-heads and sequences serially, attention.py:450)."""
    if rank != 0:
        return
    import torch

    try:
        _import_reference()
        from multipole_attn import attention as RA
        from multipole_attn import clustering as RC
        from multipole_attn.core import EngineConfig as REngineConfig
        from multipole_attn.core import HeadLayout as RHeadLayout
        kind = "reference"
    except Exception:  # baseline/_ref absent: time the pinned oracle restatement instead
        return reference_arm_port(args, rank, world)

    lay, _ = workload_cfg(args)
    cfg = REngineConfig(token_budget=args.budget, tokens_per_centroid=16, rope_theta=1e6, seed=0)
    one = RHeadLayout(lay.group_size, 1, lay.head_dim)
    ctx = args.ctx
    keys, values, qs, data = _ledger0_inputs(args, lay)
    t0 = time.perf_counter()
    led = RC.build_prefill_index_head(keys, values, ctx, cfg, 0)
    prefill_s = time.perf_counter() - t0
    n_led = args.batch * lay.num_kv_heads
    step = lambda t: RA.decode_step_attention(qs[t % len(qs)], [led], [keys], [values], ctx, t, cfg, one)
    for t in range(max(1, min(3, args.warmup))):
        step(t)
    samples = []
    for t in range(args.steps):
        t1 = time.perf_counter()
        step(args.warmup + t)
        samples.append(time.perf_counter() - t1)
        if sum(samples) > 60:
            break
    per_ledger = float(np.mean(samples))
    us = per_ledger * n_led * 1e6
    cores = _blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": us, "unit": "us/step", "n_gpus": world,
        "steps": len(samples), "warmup": args.warmup, "ms_per_step": us / 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": data,
        "config": {"workload": workload_label(args, 1), "batch": args.batch, "ctx": ctx, "budget": args.budget},
        "extrapolated": {"measured": "1 sequence x 1 kv-head ledger (4 q-heads)", "scaled_by": n_led,
                         "why": "the reference loops kv-heads and sequences serially (attention.py:450); the "
                                "whole batch would take minutes per step on the host"},
        "cpu_baseline": {"value": us, "unit": "us/step", "cores": cores, "kind": kind,
                         "sample": f"{len(samples)} reference decode_step_attention calls on 1 sequence x 1 "
                                   f"kv-head (4 q-heads), ledger from the reference build_prefill_index_head "
                                   f"in {prefill_s:.1f}s; scaled x{n_led} ledgers (the reference loops "
                                   "kv-heads / sequences serially)"},
        "e2e": {"value": us, "unit": "us/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _ledger0_inputs(args, lay):
    """Keys / values of ledger (sequence 0, kv-head 0) and its queries, drawn exactly as our arm
    draws them (bench.build_engine: the CUDA generator seeded 1000 + rank, every sequence's K then V,
    then the queries) when a GPU is present, so both arms time the same data."""
    import torch

    b, ctx, d, Hkv, Hq, G = args.batch, args.ctx, lay.head_dim, lay.num_kv_heads, lay.num_q_heads, lay.group_size
    if torch.cuda.is_available():
        dev = torch.device("cuda", 0)
        gen = torch.Generator(device=dev).manual_seed(1000)
        keys = values = None
        for s in range(b):
            k = torch.randn(1, Hkv, ctx, d, generator=gen, device=dev)
            v = torch.randn(1, Hkv, ctx, d, generator=gen, device=dev)
            if s == 0:
                # the GPU arm stores bf16 keys / values: the reference gets the same (exact in fp64) values
                keys = k[0, 0].to(torch.bfloat16).double().cpu().numpy()
                values = v[0, 0].to(torch.bfloat16).double().cpu().numpy()
            del k, v
        total = max(3, args.warmup) + args.steps + CALIB_STEPS
        Q = torch.randn(total + args.steps, b, Hq, d, generator=gen, device=dev)
        qs = Q[:, 0, :G].double().cpu().numpy()
        return keys, values, qs, ("synthetic N(0,1) Q/K/V: sequence 0 / kv-head 0 of the GPU arm's data (same "
                                  "generator and draw order, keys / values as stored in bf16)")
    gen = torch.Generator().manual_seed(0)
    keys = torch.randn(ctx, d, generator=gen).double().numpy()
    values = torch.randn(ctx, d, generator=gen).double().numpy()
    qs = torch.randn(args.steps + args.warmup, G, d, generator=gen).double().numpy()
    return keys, values, qs, "synthetic N(0,1) Q/K/V (CPU generator: no GPU to reproduce the GPU arm's draw)"


def reference_arm_port(args, rank, world):
    """--impl reference without baseline/_ref: the oracle port (pinned bit-exact to the reference
    by tests/test_golden_oracle.py) on one ledger, scaled to the batch."""
    import torch

    from oracle import mpa_oracle as O

    lay, cfg = workload_cfg(args)
    ctx = args.ctx
    keys, values, qs, data = _ledger0_inputs(args, lay)
    t0 = time.perf_counter()
    led = O.prefill_ledger(keys, values, ctx, cfg, 0)
    prefill_s = time.perf_counter() - t0
    n_led = args.batch * lay.num_kv_heads
    one = HeadLayout1(lay)
    for t in range(max(1, min(3, args.warmup))):
        O.decode_step(qs[t], [led], [keys], [values], ctx, t, cfg, one)
    samples = []
    for t in range(args.steps):
        t1 = time.perf_counter()
        O.decode_step(qs[(args.warmup + t) % len(qs)], [led], [keys], [values], ctx, t, cfg, one)
        samples.append(time.perf_counter() - t1)
        if sum(samples) > 60:
            break
    us = float(np.mean(samples)) * n_led * 1e6
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": us, "unit": "us/step", "n_gpus": world,
        "steps": len(samples), "warmup": args.warmup, "ms_per_step": us / 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": data,
        "config": {"workload": workload_label(args, 1), "batch": args.batch, "ctx": ctx, "budget": args.budget},
        "extrapolated": {"measured": "1 sequence x 1 kv-head ledger (4 q-heads)", "scaled_by": n_led},
        "cpu_baseline": {"value": us, "unit": "us/step", "cores": _blas_threads(), "kind": "port",
                         "sample": f"{len(samples)} oracle decode steps of 1 sequence x 1 kv-head (baseline/_ref "
                                   f"absent), ledger built in {prefill_s:.1f}s; scaled x{n_led} ledgers"},
        "e2e": {"value": us, "unit": "us/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def _blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        return int(max(n)) if n else 1
    except Exception:
        return os.cpu_count() or 1


def HeadLayout1(lay):
    from paper_2506_13059_b200.core import HeadLayout

    return HeadLayout(lay.group_size, 1, lay.head_dim)


def build_engine(args, rank, dev):
    """The bench workload: b sequences of ctx synthetic N(0,1) tokens written to the cache and
    indexed by the GPU clustering path; returns (engine, Q, K_new, V_new, prefill seconds)."""
    import torch

    from paper_2506_13059_b200.engine import DecodeEngine

    lay, cfg = workload_cfg(args)
    b, ctx, d = args.batch, args.ctx, lay.head_dim
    total_steps = max(3, args.warmup) + args.steps + CALIB_STEPS
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    # timed steps, then the e2e warm pass and timed pass (3 x steps), the online-update events
    tcap = ctx + 3 * total_steps + 3 * cfg.local_buffer + 8
    ps = getattr(args, "page_size", None)
    eng = DecodeEngine(cfg, lay, b, tcap=tcap, dtype=torch.bfloat16, device=dev, page_size=ps,
                       page_order="shuffled")
    if ps:
        eng.reserve(ctx)  # the prompt's pages
    for s in range(b):  # prompt KV, one sequence at a time to bound temporaries
        k = torch.randn(1, lay.num_kv_heads, ctx, d, generator=gen, device=dev)
        v = torch.randn(1, lay.num_kv_heads, ctx, d, generator=gen, device=dev)
        _write_seq(eng, s, k, v)
        del k, v
    eng.cache_len[:] = ctx
    eng._sync_scalars()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.prefill()
    torch.cuda.synchronize()
    prefill_s = time.perf_counter() - t0
    n = total_steps + args.steps
    Q = torch.randn(n, b, lay.num_q_heads, d, generator=gen, device=dev)
    KN = torch.randn(n, b, lay.num_kv_heads, d, generator=gen, device=dev)
    VN = torch.randn(n, b, lay.num_kv_heads, d, generator=gen, device=dev)
    return eng, Q, KN, VN, prefill_s


# ---------------------------------------------------------------------------- GPU arm


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if world > 1 and rank != 0:
            return
        reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.workload != "c2":
        args.no_cpu = True  # the CPU side-by-side is quoted on the metric's config (c2)
    if args.workload == "c5" and world > 1:
        return main_sharded(args, rank, world, local)

    def barrier():
        if world > 1:
            dist.barrier()

    from paper_2506_13059_b200 import clustering
    from paper_2506_13059_b200._lib import lib as _load_lib
    from paper_2506_13059_b200.engine import DecodeEngine
    from paper_2506_13059_b200.roofline import decode_bytes, dense_bytes

    _load_lib()
    lay, cfg = workload_cfg(args)
    b, ctx, d, G = args.batch, args.ctx, lay.head_dim, lay.group_size
    W, K = max(3, args.warmup), args.steps
    dev = torch.device("cuda", local)
    eng, Q, KN, VN, prefill_s = build_engine(args, rank, dev)
    import gc
    gen = torch.Generator(device=dev).manual_seed(2000 + rank)
    total_steps = W + K
    flush = L2Flush(dev)
    stream = torch.cuda.current_stream()

    def timed(fn, n, *, start=0):
        evs = []
        for i in range(n):
            flush(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(start + i)
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return [a.elapsed_time(c) for a, c in evs]  # ms

    # ---- warmup + timed multipole steps (attend + append)
    for i in range(W):
        eng.step(Q[i], KN[i], VN[i])
    torch.cuda.synchronize()
    barrier()
    with Clocks(local) as clk:
        # keep the GPU loaded (attention only, no state change) until the sampler has seen it
        # busy, then time the K steps; the sampler runs across both
        t_end = time.perf_counter() + (0.0 if args.profile else 1.5)
        while time.perf_counter() < t_end:
            for _ in range(20):
                eng.attend(Q[0])
            torch.cuda.synchronize()
        # setup garbage collected now and the long-lived objects frozen, so a generation-2
        # collection does not land inside a (host-driven) online update of the timed steps
        gc.collect()
        gc.freeze()
        barrier()
        step_ms = timed(lambda i: eng.step(Q[i], KN[i], VN[i]), K, start=W)
        torch.cuda.synchronize()
        barrier()
        t_end = time.perf_counter() + (0.0 if args.profile else 0.5)
        while time.perf_counter() < t_end:
            for _ in range(20):
                eng.attend(Q[0])
            torch.cuda.synchronize()
    stats = eng.head_stats()
    scored = (eng.led.n_fine.copy() if cfg.hierarchy is None
              else eng.led.n_coarse + eng.n_cand.cpu().numpy().astype(np.int64))
    ms_step = float(np.mean(step_ms))

    # ---- fused decode kernel (dominant kernel) for the roofline: alone (L2 flushed, its lists cold
    # too) and in the step chain (lookup launch, then events around the fused kernel on the engine
    # stream -- its work lists come warm from the lookup as inside the step graph)
    one_kernel = False
    eng.rotate(Q[0], exact=True, lookup=False)
    eng.lookup(Q[0])
    torch.cuda.synchronize()
    fstats = eng.head_stats()
    fused_ms = timed(lambda i: eng.fused(), K)
    fev = []
    for i in range(K):
        flush(i)
        if not eng.fused_lookup_path():
            eng.rotate(Q[i], exact=True, lookup=False)
        eng.lookup(Q[i])
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.fused()
        z.record(stream)
        fev.append((a, z))
    torch.cuda.synchronize()
    fused_step_avg = float(np.mean([a.elapsed_time(z) for a, z in fev]))
    lookup_ms = timed(lambda i: eng.lookup(Q[0]), K)  # the lookup launch(es): views + logits + select + lists
    nbytes = decode_bytes(fstats, scored, d, G, 2)
    kernel_bytes = nbytes["fused"]
    fused_avg = float(np.mean(fused_ms))

    # ---- dense decode comparator (same cache, same kernel family, tok == NULL)
    for i in range(3):
        eng.attend_dense(Q[i])
    dense_ms = timed(lambda i: eng.attend_dense(Q[i]), K)
    dense_avg = float(np.mean(dense_ms))
    dbytes = dense_bytes(np.repeat(eng.cache_len, lay.num_kv_heads), d, G, 2)
    fi_ms = None if (args.profile or eng.block_table is not None) else flashinfer_dense(eng, Q[0], K, timed)

    # ---- end to end through the public API from pinned host buffers
    qh = Q[total_steps:total_steps + K].cpu().pin_memory()
    kh = KN[total_steps:total_steps + K].cpu().pin_memory()
    vh = VN[total_steps:total_steps + K].cpu().pin_memory()
    oh = torch.empty(b, lay.num_q_heads, d, dtype=torch.float32).pin_memory()
    for i in range(K):  # warm-up pass over the same host buffers (a server reuses its pinned staging)
        eng.step_host(qh[i], kh[i], vh[i], oh)
    torch.cuda.synchronize()
    e2e_ms = timed(lambda i: eng.step_host(qh[i], kh[i], vh[i], oh), K)
    _ = oh.sum().item()
    e2e_avg = float(np.mean(e2e_ms))
    h2d = (qh[0].numel() + kh[0].numel() + vh[0].numel()) * 4
    d2h = oh.numel() * 4
    dropin = None if (args.profile or args.workload != "c2" or world > 1) else dropin_step(args, lay, cfg, K)

    # ---- online cluster update events (C4-style overhead, amortised over L steps): the first one
    # in the process also pays one-time lazy CUDA module loads, so two events run and the second,
    # steady-state one is reported (the first is listed beside it)
    L = cfg.local_buffer
    upd, update_ms, update_first_ms = {"rounds": 0}, 0.0, 0.0
    for ev in range(0 if args.profile else 2):
        need = int(2 * L - (eng.cache_len[0] - eng.buffer_start[0]))
        if need > 0:
            eng.write_tokens(torch.randn(b, lay.num_kv_heads, need, d, generator=gen, device=dev),
                             torch.randn(b, lay.num_kv_heads, need, d, generator=gen, device=dev))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        upd = clustering.online_update(eng, list(range(b)), eng.cursor + ev)
        torch.cuda.synchronize()
        update_first_ms, update_ms = update_ms, (time.perf_counter() - t0) * 1e3

    # ---- max over ranks
    vals = torch.tensor([ms_step, e2e_avg, fused_avg, dense_avg, fused_step_avg or fused_avg], device=dev,
                        dtype=torch.float64)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms_step, e2e_avg, fused_avg, dense_avg, fused_step_avg = (float(x) for x in vals.cpu())

    if rank == 0:
        hbm, peak_kind = peaks()
        achieved = kernel_bytes / (fused_step_avg * 1e-3) / 1e9
        traffic = load_traffic(args.workload, b)
        line = {
            "metric": METRIC,
            "value": ms_step * 1e3,
            "unit": "us/step",
            "n_gpus": world,
            "steps": K,
            "warmup": W,
            "ms_per_step": ms_step,
            "higher_is_better": False,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic N(0,1) Q/K/V (random-init Qwen3-8B attention shape), seed 1000+rank",
            "config": {"workload": workload_label(args, world), "batch": b, "ctx": ctx,
                       "budget": args.budget, "tokens_per_centroid": cfg.fine_ratio,
                       "l2": L2Flush.DESC,
                       "kv_cache": (f"paged: {args.page_size}-token pages in shuffled order, HND pools"
                                    if args.page_size else "flat [L, tcap, d]"),
                       "parallelism": f"batch-sharded replicas x{world}"},
            "speedup_vs_dense": dense_avg / ms_step,
            "dense_us_per_step": dense_avg * 1e3,
            "dense_gbs": dbytes / (dense_avg * 1e-3) / 1e9,
            "flashinfer_dense_us": (fi_ms * 1e3) if fi_ms else None,
            "sequences_per_s": world * b / (ms_step * 1e-3),
            "roofline": {"bound": "hbm",
                         "kernel": ("mpa_decode_step (step_kernel: lookup + selection + replacement + exact "
                                    "attention, one launch per step)") if one_kernel
                         else "mpa_sparse_decode (decode_sk_kernel)",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "peak_kind": peak_kind, "traffic": traffic,
                         "algorithmic_bytes_per_launch": kernel_bytes, "launch_us": fused_step_avg * 1e3,
                         "timing": ("CUDA events around the step kernel launched alone on the engine stream, "
                                    "L2 flushed before every launch") if one_kernel
                         else ("CUDA events around the fused kernel in the step chain (engine stream, "
                               "lists warm from the selection), L2 flushed before every step"),
                         "launch_us_alone_cold": fused_avg * 1e3},
            "step_roofline": {"bytes": nbytes["step"], "GBs": nbytes["step"] / (ms_step * 1e-3) / 1e9,
                              "frac": nbytes["step"] / (ms_step * 1e-3) / 1e9 / hbm,
                              "lookup_us": float(np.mean(lookup_ms)) * 1e3},
            "selection": {"mean_exact_tokens": float(fstats[:, 0].mean()),
                          "mean_rejected_centroids": float(fstats[:, 1].mean()),
                          "mean_scored_centroids": float(np.mean(scored)),
                          "memop_ratio": nbytes["step"] / dbytes},
            # the slowest timed steps (with an online update inside, they show the update's cost)
            "step_ms_top": sorted((round(float(x), 3) for x in step_ms), reverse=True)[:6],
            "step_ms_median": float(np.median(step_ms)),
            "update": {"ms_per_event": update_ms, "first_event_ms": update_first_ms,
                       "amortized_us_per_step": update_ms * 1e3 / L,
                       "pct_of_step": update_ms / L / ms_step * 100.0, "lloyd_rounds": upd["rounds"],
                       "prefill_s": prefill_s},
            "e2e": {"value": e2e_avg * 1e3, "unit": "us/step", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "median_us": float(np.median(e2e_ms)) * 1e3,
                    "top_us": sorted((round(float(x) * 1e3, 1) for x in e2e_ms), reverse=True)[:5],
                    "api": "engine.DecodeEngine.step_host (batched public API, pinned host buffers)"},
            "e2e_dropin": dropin,
            "graph_captures": eng.n_captures,
            # per step: the step graph (flat bf16 path: lookup + append, fused decode -- reading the
            # step's q / k / v in place; else input staging + 2 rotations, logits, select+lists,
            # fused decode, append)
            "gpu_launches": (2 if eng._graph_raw is not None else 3 if eng.fused_lookup_path() else 7) * K,
            "clocks": clk.summary(),
        }
        if not args.no_cpu and not args.profile:
            line["cpu_baseline"] = cpu_leg(eng, lay, cfg, Q, b)
        print(json.dumps(line), flush=True)
    barrier()
    if world > 1:
        dist.destroy_process_group()


def main_sharded(args, rank, world, local):
    """C5 at N > 1: one 128K context per sequence, KV blocks sharded over the ranks
    (paper_2506_13059_b200/sharded.py); three NCCL all-gathers per step; strong scaling."""
    import torch
    import torch.distributed as dist

    from paper_2506_13059_b200._lib import lib as _load_lib
    from paper_2506_13059_b200.sharded import ShardedDecodeEngine, TorchComm

    _load_lib()
    lay, cfg = workload_cfg(args)
    b, ctx, d = args.batch, args.ctx, lay.head_dim
    W, K = max(3, args.warmup), args.steps
    dev = torch.device("cuda", local)
    comm = TorchComm()
    gen = torch.Generator(device=dev).manual_seed(1000)  # identical prompt / queries on every rank
    tcap = ctx + 2 * (W + 2 * K) + 3 * cfg.local_buffer + 8
    se = ShardedDecodeEngine(cfg, lay, b, tcap, rank, world, dtype=torch.bfloat16, device=dev)
    eng = se.eng
    for s_ in range(b):
        k = torch.randn(1, lay.num_kv_heads, ctx, d, generator=gen, device=dev)
        v = torch.randn(1, lay.num_kv_heads, ctx, d, generator=gen, device=dev)
        _write_seq(eng, s_, k, v)
        del k, v
    eng.cache_len[:] = ctx
    eng._sync_scalars()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    se.prefill_local()
    n_all = comm.all_gather(torch.as_tensor(eng.led.n_fine, dtype=torch.int64, device=dev)).cpu().numpy()
    se.set_gid_offsets(n_all)
    torch.cuda.synchronize()
    prefill_s = time.perf_counter() - t0
    n = W + 2 * K
    Q = torch.randn(n, b, lay.num_q_heads, d, generator=gen, device=dev)
    KN = torch.randn(n, b, lay.num_kv_heads, d, generator=gen, device=dev)
    VN = torch.randn(n, b, lay.num_kv_heads, d, generator=gen, device=dev)
    flush = L2Flush(dev)
    stream = torch.cuda.current_stream()

    # the whole sharded step (local kernels + the three NCCL all-gathers) as one CUDA graph, checked
    # against the eager step once; any failure keeps the eager path
    def agree(ok: bool) -> bool:  # every rank, or none
        t = torch.tensor([1.0 if ok else 0.0], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item() == 1.0)

    graphed = False
    if dist.get_backend() == "nccl":
        try:  # the capture itself runs no collective, so a rank failing here leaves the others in step
            se.capture_attend(Q[0], comm)
            ok = True
        except Exception:
            ok = False
        if agree(ok):
            want = se.attend(Q[0], comm).clone()
            got = se.attend_graphed(Q[0], comm).clone()
            graphed = agree(torch.equal(got, want))

    def step(i):
        out = se.attend_graphed(Q[i], comm) if graphed else se.attend(Q[i], comm)
        eng.write_tokens(KN[i][:, :, None], VN[i][:, :, None])
        return out

    def timed(fn, count, start=0):
        evs = []
        for i in range(count):
            flush(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(start + i)
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return [a.elapsed_time(c) for a, c in evs]

    for i in range(W):
        step(i)
    torch.cuda.synchronize()
    dist.barrier()
    with Clocks(local) as clk:
        dist.barrier()
        step_ms = timed(step, K, W)
        dist.barrier()
    # dense comparator over this rank's token range, merged across ranks the same way
    s0 = int(eng.sink_end[0])
    Wb = cfg.block_size
    n_sealed = (int(eng.buffer_start[0]) - s0) // Wb
    lo_b, hi_b = n_sealed * rank // world, n_sealed * (rank + 1) // world
    lo = 0 if rank == 0 else s0 + lo_b * Wb
    hi_fn = (lambda: int(eng.cache_len[0])) if rank == world - 1 else (lambda: s0 + hi_b * Wb)
    ids = torch.arange(lo, hi_fn(), dtype=torch.int32, device=dev)
    tokd = torch.zeros(eng.L, max(1, ids.numel()), dtype=torch.int32, device=dev)
    tokd[:, : ids.numel()] = ids
    ntokd = torch.full((eng.L,), ids.numel(), dtype=torch.int32, device=dev)
    from paper_2506_13059_b200._lib import call, ptr, stream_ptr

    def dense(i):
        eng.rotate(Q[i])
        ws = eng._workspace(0)
        call("mpa_sparse_decode_partials", eng.cache_struct, ptr(eng.q_rot), eng.Hkv, eng.G, ptr(tokd), ptr(ntokd),
             tokd.shape[1], None, None, None, 0, None, 0, None, 0, 0, ptr(ws), ws.numel(), ptr(se.part), stream_ptr())
        return se.phase_merge(comm.all_gather(se.part))

    for i in range(3):
        dense(i)
    dense_ms = timed(dense, K)
    vals = torch.tensor([float(np.mean(step_ms)), float(np.mean(dense_ms))], device=dev, dtype=torch.float64)
    dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms_step, dense_avg = (float(x) for x in vals.cpu())
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": ms_step * 1e3, "unit": "us/step", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_step, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic N(0,1) Q/K/V (random-init Qwen3-8B attention shape)",
            "config": {"workload": workload_label(args, world), "batch": b, "ctx": ctx, "budget": args.budget,
                       "parallelism": f"KV-sequence-sharded x{world} (NCCL all-gather of (M,Z), candidate "
                                      "prefixes and (m,s,a) partials)",
                       "step_graph": "one CUDA graph per step incl. the NCCL all-gathers" if graphed else "eager",
                       "l2": L2Flush.DESC},
            "speedup_vs_dense": dense_avg / ms_step, "dense_us_per_step": dense_avg * 1e3,
            "sequences_per_s": b / (ms_step * 1e-3), "prefill_s": prefill_s,
            "gpu_launches": 12 * K, "clocks": clk.summary(),
        }), flush=True)
    dist.barrier()
    dist.destroy_process_group()


class L2Flush:
    """Between timed steps: write a 256 MB buffer (evicts everything; L2 > 126 MB), then read
    another 256 MB one, so the step starts with a cold L2 that holds no dirty lines -- the write
    flush alone would charge the step for writing back 126 MB of the flush buffer."""

    DESC = "flushed before every timed step (256 MB write, then 256 MB read: cold and clean)"

    def __init__(self, dev):
        import torch

        self.w = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
        self.r = torch.zeros(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
        self.acc = torch.zeros((), dtype=torch.float32, device=dev)

    def __call__(self, i):
        self.w.fill_(float(i))
        self.acc += self.r.sum()


def dropin_step(args, lay, cfg, K):
    """The reference's own call, paper_2506_13059_b200.step(state, q, k, v) (pipeline.py:124): one
    sequence (its signature has no batch) of the workload's shape and context, bf16 serving cache,
    numpy inputs in, fp64 outputs + the DecodeReport (selected refs / tokens per head) out, timed by
    wall clock around each call (every call ends with its host reads)."""
    import torch

    import paper_2506_13059_b200 as mpa

    ctx, d = args.ctx, lay.head_dim
    n = ctx + K + 4
    g = torch.Generator(device="cuda").manual_seed(7)
    keys = torch.randn(lay.num_kv_heads, n, d, generator=g, device="cuda").cpu().numpy()
    values = torch.randn(lay.num_kv_heads, n, d, generator=g, device="cuda").cpu().numpy()
    queries = torch.randn(lay.num_q_heads, K + 4, d, generator=g, device="cuda").cpu().numpy()
    trace = mpa.KvTrace(lay, ctx, keys, values, queries)
    state = mpa.prefill(trace, cfg, dtype=torch.bfloat16)
    ms = []
    for t in range(K + 3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mpa.step(state, queries[:, t], keys[:, ctx + t], values[:, ctx + t])
        if t >= 3:
            ms.append((time.perf_counter() - t0) * 1e3)
    del state
    torch.cuda.empty_cache()
    return {"value": float(np.mean(ms)) * 1e3, "unit": "us/step", "batch": 1,
            "api": "paper_2506_13059_b200.step(state, q, k, v) -- the reference's pipeline.step signature "
                   "(one sequence, numpy in, fp64 outputs + DecodeReport out), bf16 cache, wall clock",
            "h2d_bytes_per_step": int((lay.num_q_heads + 2 * lay.num_kv_heads) * d * 4),
            "d2h_bytes_per_step": int(lay.num_q_heads * d * 4)}


def _write_seq(eng, s, k, v):
    """Write one sequence's prompt K/V (fp32 [1, Hkv, n, d]) into its ledger rows at position 0."""
    import torch

    from paper_2506_13059_b200._lib import MpaCache, call, dtype_code, ptr, stream_ptr

    Hkv = eng.Hkv
    n = k.shape[2]
    if eng.block_table is None:
        sub = MpaCache(ptr(eng.k_rot[s * Hkv]), ptr(eng.k_raw[s * Hkv]), ptr(eng.v[s * Hkv]), dtype_code(eng.dtype),
                       Hkv, eng.tcap, eng.d)
    else:  # the page pools with sequence s's block-table row
        sub = MpaCache(ptr(eng.k_rot), ptr(eng.k_raw[s * Hkv]), ptr(eng.v), dtype_code(eng.dtype), Hkv, eng.tcap,
                       eng.d, ptr(eng.block_table[s]), eng.page_size, eng.pages_per_seq, eng.n_pages, Hkv)
    pos0 = torch.zeros(Hkv, dtype=torch.int32, device=eng.device)
    kk = k.reshape(Hkv, n, eng.d).contiguous()
    vv = v.reshape(Hkv, n, eng.d).contiguous()
    call("mpa_kv_write", sub, ptr(kk), ptr(vv), ptr(pos0), n, ptr(eng.inv_freq), stream_ptr())
    torch.cuda.synchronize()


def flashinfer_dense(eng, q, K, timed):
    """Cross-check of the dense comparator with flashinfer's decode (pre-rotated K), if usable."""
    try:
        import flashinfer  # noqa: F401
        import torch

        kc = eng.k_rot[:eng.Hkv, : int(eng.cache_len[0])].transpose(0, 1).contiguous()
        vc = eng.v[:eng.Hkv, : int(eng.cache_len[0])].transpose(0, 1).contiguous()
        qq = eng.q_rot[0].to(torch.bfloat16) * math.sqrt(eng.d)
        flashinfer.single_decode_with_kv_cache(qq, kc, vc, kv_layout="NHD")
        ms = timed(lambda i: flashinfer.single_decode_with_kv_cache(qq, kc, vc, kv_layout="NHD"), K)
        return float(np.mean(ms)) * eng.n_seq  # batch = n_seq independent sequences
    except Exception:
        return None


def load_traffic(workload, batch):
    """dram read+write bytes per decode_sk_kernel launch from the committed ncu --set full capture,
    only when that capture was taken on this workload (else null)."""
    p = os.path.join(ROOT, "profiles", "fused_traffic.json")
    try:
        with open(p) as fh:
            rec = json.load(fh)
        if rec.get("workload") == workload and int(rec.get("batch", -1)) == batch:
            return rec.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


def reference_cpu_time(keys, values, qs, ctx, budget, group, d, n_steps=3):
    """Seconds per decode step of ONE ledger (1 sequence x 1 kv-head, its G q-heads) through the
    real reference (baseline/_ref): ledger from build_prefill_index_head, steps through
    decode_step_attention, plus one dense exact_attention pass (the reference's oracle mode)
    over the same ledger.  Returns None if the reference is not importable."""
    try:
        _import_reference()
        from multipole_attn import attention as RA
        from multipole_attn import clustering as RC
        from multipole_attn.core import EngineConfig as REngineConfig
        from multipole_attn.core import HeadLayout as RHeadLayout
        from multipole_attn.rope import RopeParams
    except Exception:
        return None
    cfg = REngineConfig(token_budget=budget, tokens_per_centroid=16, rope_theta=1e6, seed=0)
    one = RHeadLayout(group, 1, d)
    t0 = time.perf_counter()
    led = RC.build_prefill_index_head(keys, values, ctx, cfg, 0)
    prefill_s = time.perf_counter() - t0
    RA.decode_step_attention(qs[0], [led], [keys], [values], ctx, 0, cfg, one)
    t0 = time.perf_counter()
    for t in range(n_steps):
        RA.decode_step_attention(qs[t % len(qs)], [led], [keys], [values], ctx, t, cfg, one)
    sparse = (time.perf_counter() - t0) / n_steps
    params = RopeParams(head_dim=d, theta=cfg.rope_theta, window_offset=cfg.window_offset)
    pos = np.arange(ctx, dtype=np.int64)
    t0 = time.perf_counter()
    for g in range(group):
        RA.exact_attention(qs[0][g], ctx, keys, values, pos, params)
    dense = time.perf_counter() - t0
    return {"sparse_s": sparse, "dense_s": dense, "prefill_s": prefill_s, "steps": n_steps}


def cpu_leg(eng, lay, cfg, Q, b):
    """cpu_baseline: the reference package itself (baseline/_ref) on one ledger of the bench
    workload (sequence 0, kv-head 0: the same keys / values / queries the GPU sees), scaled to
    the batch; the numpy oracle restatement with the GPU-built ledger if the reference is absent."""
    n = int(eng.cache_len[0])
    keys = eng.k_raw[0, :n].float().cpu().numpy()
    vals = eng.v[0, :n].float().cpu().numpy()
    qs = [Q[i, 0, :lay.group_size].cpu().numpy() for i in range(3)]
    n_led = b * lay.num_kv_heads
    r = reference_cpu_time(keys, vals, qs, n, cfg.token_budget, lay.group_size, lay.head_dim)
    if r is not None:
        return {"value": r["sparse_s"] * n_led * 1e6, "unit": "us/step", "cores": _blas_threads(),
                "kind": "reference",
                "sample": f"{r['steps']} reference decode_step_attention calls on 1 sequence x 1 kv-head "
                          f"(4 q-heads) of the bench workload (ledger by the reference prefill in "
                          f"{r['prefill_s']:.1f}s), scaled x{n_led} ledgers; the reference dense oracle of "
                          f"the same ledger scales to {r['dense_s'] * n_led * 1e6:.0f} us/step"}
    from tests.bridge import to_oracle

    led = to_oracle(eng.export_ledger(0))
    led.total = n
    sparse_s, dense_s = cpu_oracle_time(lay, cfg, keys, vals, qs, led, n)
    return {"value": sparse_s * n_led * 1e6, "unit": "us/step", "cores": 1, "kind": "port",
            "sample": "3 oracle decode steps of 1 sequence x 1 kv-head (4 q-heads) at the bench config, scaled "
                      f"x{n_led} ledgers; dense oracle of the same ledger {dense_s * n_led * 1e6:.0f} us/step"}


if __name__ == "__main__":
    main()
