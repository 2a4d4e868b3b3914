"""GPU key clustering: blockwise prefill index, online update, sliding-window split/settle and
the two-level hierarchy, driving the batched k-means kernels of libmpattn (csrc/mpa_cluster.cu).

Reference (pkg/src/multipole_attn/clustering.py):
  build_prefill_index_head  :288-326   -> prefill_ledgers()
  append_tokens             :404-472   -> online_update()
  _split_final / _settle    :343-401   -> _split()
  build_hierarchy           :210-264   -> _hierarchy()
  kmeans / lloyd            :123-184   -> KMeansBatch (all problems of a call in one batch)

The module also carries the reference's module-level API (names, arguments, types, exceptions of
clustering.py:33-657: Cluster / Block / BlockLedger, kmeans, lloyd, build_prefill_index(_head),
append_tokens, build_hierarchy, the positional comparator, audit_ledger, wcss, the JSON dump) for
callers holding numpy arrays; each routes through the same kernels (a one-ledger engine, or the
fp64 kernels of csrc/mpa_refapi.cu), see the end of this file.

Everything numerical runs on the GPU.  The host only draws the reference's RNG indices
(numpy PCG64 with the same seeds: block k-means init, update samples, hierarchy init), keeps
the per-ledger block table (spans and cluster counts) and sizes the problem batches.
"""

from __future__ import annotations

import numpy as np
import torch

from ._lib import MpaKm, call, dtype_code, ptr, stream_ptr
from .core import ConfigError, block_seed, update_rng
from .ledger import BlockRow

MAX_POINTS = 16384  # per problem (csrc/mpa_cluster.cu kMaxPoints)


def _scratch(cache, name: str, numel: int, dtype, device) -> torch.Tensor:
    """A flat scratch tensor of >= numel elements kept in `cache` between calls and grown by 1.5x, so
    the online updates (whose problem sizes creep up event by event) reuse the same device blocks
    instead of asking the allocator for slightly larger ones every time (cudaMalloc stalls)."""
    if cache is None:
        return torch.empty(max(numel, 1), dtype=dtype, device=device)
    t = cache.get(name)
    if t is None or t.numel() < numel or t.dtype != dtype:
        t = torch.empty(max(int(numel * 1.5), 1), dtype=dtype, device=device)
        cache[name] = t
    return t[: max(numel, 1)]


class KMeansBatch:
    """One batch of independent Lloyd problems (l, start, n, k) on a shared point source."""

    def __init__(self, device, d: int, probs, init: torch.Tensor, *, pts=None, tcap: int = 0, pts64=None, wts=None,
                 rows64_cap: int = 0, min_iters: int = 0, count_init: torch.Tensor | None = None, cache=None):
        arr = np.asarray(probs, np.int64).reshape(-1, 4)
        self.probs = arr
        self.P = arr.shape[0]
        n, k = arr[:, 2], arr[:, 3]
        if self.P and int(n.max()) > MAX_POINTS:
            raise ConfigError(f"k-means problem with {int(n.max())} points > {MAX_POINTS} per problem")
        self.pt_off = np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64)
        self.c_off = np.concatenate([[0], np.cumsum(k)[:-1]]).astype(np.int64)
        i32 = dict(dtype=torch.int32, device=device)
        N, K = int(n.sum()), int(k.sum())
        self.d = d
        # the six per-problem tables in one host -> device copy
        names = ("l", "start", "n", "k", "pt_off", "c_off")
        tab = torch.as_tensor(np.stack([arr[:, 0], arr[:, 1], n, k, self.pt_off, self.c_off]).astype(np.int32)
                              if self.P else np.zeros((6, 1), np.int32), **i32)
        self.t = {name: tab[i] for i, name in enumerate(names)}
        sc = lambda name, n, dt: _scratch(cache, name, n, dt, device)
        # every Lloyd kernel writes these before reading them (the assignment is zeroed for
        # callers that read it before a pass)
        self.assign = sc("assign", N, torch.int32).zero_()
        self.prev = sc("prev", N, torch.int32)
        self.p2 = sc("p2", N, torch.float64)
        self.order = sc("order", N, torch.int32)
        self.cent = init.to(torch.float64).contiguous().reshape(-1, d)
        assert self.cent.shape[0] == K, (self.cent.shape, K)
        self.c2 = torch.zeros(max(K, 1), dtype=torch.float64, device=device)
        self.count = (count_init.to(torch.int32).contiguous() if count_init is not None
                      else torch.zeros(max(K, 1), **i32))
        self.cstart = torch.zeros(max(K, 1), **i32)
        self.dirty = sc("dirty", K, torch.int32)
        self.state = torch.zeros(max(self.P, 1), 4, **i32)
        self.flag = torch.zeros(2, **i32)
        self.src = (pts, tcap, pts64, wts, rows64_cap)
        self.min_iters = min_iters
        self.n_max = int(n.max()) if self.P else 0
        self.k_max = int(k.max()) if self.P else 0
        self.sum_n, self.sum_k = N, K
        # tcgen05 assignment (csrc/mpa_km_tc.cu) for bf16 key sources with d = 128
        self.pts_rows = int(pts.shape[0] * pts.shape[1]) if pts is not None else 0
        self.tc_ws = None
        if pts is not None and pts.dtype == torch.bfloat16 and d == 128 and self.P:
            from ._lib import lib

            nb = int(lib().mpa_km_tc_workspace(self.P, K, N, d))
            self.tc_ws = _scratch(cache, "tc_ws", nb, torch.uint8, device)

    def struct(self) -> MpaKm:
        pts, tcap, pts64, wts, rcap = self.src
        t = self.t
        return MpaKm(self.P, self.d, ptr(pts), dtype_code(pts.dtype) if pts is not None else 0, tcap, ptr(pts64),
                     ptr(wts), rcap, self.n_max, self.k_max, self.min_iters, ptr(t["l"]), ptr(t["start"]),
                     ptr(t["n"]), ptr(t["k"]), ptr(t["pt_off"]), ptr(t["c_off"]), ptr(self.assign), ptr(self.prev),
                     ptr(self.p2), ptr(self.cent), ptr(self.c2), ptr(self.count), ptr(self.order), ptr(self.cstart),
                     ptr(self.state), ptr(self.flag), self.pts_rows, self.sum_n, self.sum_k, ptr(self.tc_ws),
                     self.tc_ws.numel() if self.tc_ws is not None else 0, ptr(self.dirty))

    def lloyd(self) -> int:
        import ctypes

        r = ctypes.c_int32(0)
        call("mpa_km_lloyd", self.struct(), ctypes.byref(r), stream_ptr())
        return int(r.value)

    def means(self) -> None:
        call("mpa_km_means", self.struct(), stream_ptr())

    def nonempty(self) -> np.ndarray:
        nk = torch.zeros(max(self.P, 1), dtype=torch.int32, device=self.assign.device)
        call("mpa_km_count_nonempty", self.struct(), ptr(nk), stream_ptr())
        self.nk = nk[: self.P].cpu().numpy().astype(np.int64)
        return self.nk

    def counts(self, p: int) -> torch.Tensor:
        c0, k = int(self.c_off[p]), int(self.probs[p, 3])
        return self.count[c0:c0 + k]

    def centroids(self, p: int) -> torch.Tensor:
        c0, k = int(self.c_off[p]), int(self.probs[p, 3])
        return self.cent[c0:c0 + k]


def _i32(eng, a) -> torch.Tensor:
    # device copy of a small host index array; callers keep the tensor alive across the launch
    return torch.as_tensor(np.asarray(a), dtype=torch.int32, device=eng.device)


def _check_level_cap(km: KMeansBatch, first: np.ndarray, cap: int, what: str) -> None:
    """The level writer compacts each problem's non-empty clusters to rows [first, first + nk) of
    its ledger with no device-side bound: check them on the host before the launch."""
    nk = getattr(km, "nk", None)
    if nk is None:
        nk = km.nonempty()
    over = np.flatnonzero(np.asarray(first, np.int64) + nk > cap)
    if over.size:
        i = int(over[0])
        raise ConfigError(f"{what} cluster capacity exceeded: problem {i} writes rows "
                          f"[{int(first[i])}, {int(first[i] + nk[i])}) of {cap}")


def _write_fine(eng, km: KMeansBatch, f0: np.ndarray, mbase: np.ndarray) -> None:
    led = eng.led
    _check_level_cap(km, f0, led.kcap, "fine")
    f0_d, mb_d = _i32(eng, f0), _i32(eng, mbase)
    call("mpa_km_write_level", km.struct(), eng.cache_struct, None, ptr(f0_d), ptr(mb_d),
         ptr(led.kc64), ptr(led.vc64), ptr(led.kc), ptr(led.vc), dtype_code(led.dtype), ptr(led.size), ptr(led.off),
         ptr(led.mem), led.kcap, led.tcap, stream_ptr())


def _write_coarse(eng, km: KMeansBatch, c0: np.ndarray, mbase: np.ndarray) -> None:
    led = eng.led
    _check_level_cap(km, c0, led.ccap, "coarse")
    c0_d, mb_d = _i32(eng, c0), _i32(eng, mbase)
    call("mpa_km_write_level", km.struct(), None, ptr(led.vc64), ptr(c0_d), ptr(mb_d),
         ptr(led.ckc64), ptr(led.cvc64), ptr(led.ckc), ptr(led.cvc), dtype_code(led.dtype), ptr(led.csize),
         ptr(led.coff), ptr(led.child), led.ccap, led.kcap, stream_ptr())


def _refresh_counts(eng, ledgers) -> None:
    led = eng.led
    for l in ledgers:
        rows = led.blocks[l]
        led.n_fine[l] = rows[-1].f0 + rows[-1].fk if rows else 0
        led.n_coarse[l] = rows[-1].c0 + rows[-1].ck if rows else 0
        if led.n_fine[l] > led.kcap or led.n_coarse[l] > max(led.ccap, 0) and led.hierarchy:
            raise ConfigError(f"ledger {l}: cluster capacity exceeded (fine {led.n_fine[l]}/{led.kcap}, "
                              f"coarse {led.n_coarse[l]}/{led.ccap})")
    led.count.copy_(torch.as_tensor(led.n_fine, dtype=torch.int32))
    if led.hierarchy:
        led.ccount.copy_(torch.as_tensor(led.n_coarse, dtype=torch.int32))
    K = int(led.n_fine.max()) if led.L else 0
    if K:
        mask = torch.arange(K, device=eng.device)[None, :] < led.count[:, None]
        led.set_max_size_async((led.size[:, :K] * mask).amax(dim=1))


def _head(eng, l: int) -> int:
    """kv-head index of ledger l for the block seeds (an engine built for one reference head sets
    eng.head_ids to that head)."""
    ids = getattr(eng, "head_ids", None)
    return int(ids[l]) if ids is not None else l % eng.Hkv


# ---------------------------------------------------------------------------- prefill


def prefill_ledgers(eng, owned=None) -> None:
    """Blockwise k-means of every ledger's prompt (clustering.py:288-326); k = ceil(n / r),
    init = default_rng(block_seed(seed, head, b)).choice(n, k, replace=False).
    owned(b, n_blocks) -> bool restricts the ledger to some of its blocks (sequence sharding:
    block seeds keep their global index b, fine ids are local to the owned blocks)."""
    cfg, led = eng.cfg, eng.led
    W = cfg.block_size
    eng.set_prompt_layout()
    probs, inits, owners = [], [], []
    tables = []
    for l in range(eng.L):
        s = l // eng.Hkv
        s0, b0 = int(eng.sink_end[s]), int(eng.buffer_start[s])
        nsealed = (b0 - s0) // W
        spans = [(s0 + b * W, s0 + b * W + W) for b in range(nsealed)] + [(s0 + nsealed * W, b0)]
        if owned is not None:
            spans = [sp if owned(b, len(spans)) else None for b, sp in enumerate(spans)]
        tables.append(spans)
        for b, sp in enumerate(spans):
            if sp is None:
                continue
            lo, hi = sp
            n = hi - lo
            if n <= 0:
                continue
            k = min(max(1, -(-n // cfg.fine_ratio)), n)
            pick = np.random.default_rng(block_seed(cfg.seed, _head(eng, l), b)).choice(n, size=k, replace=False)
            probs.append((l, lo, n, k))
            inits.append(eng.k_raw[l, lo + torch.as_tensor(pick, device=eng.device)].double())
            owners.append((l, b))
    km = KMeansBatch(eng.device, eng.d, probs, torch.cat(inits) if inits else torch.zeros(0, eng.d),
                     pts=eng.k_raw, tcap=eng.tcap, min_iters=cfg.prefill_kmeans_iters)
    eng.last_lloyd_rounds = km.lloyd() if probs else 0
    nk = km.nonempty()
    f0 = np.zeros(len(probs), np.int64)
    mbase = np.zeros(len(probs), np.int64)
    per = {o: i for i, o in enumerate(owners)}
    for l in range(eng.L):
        s0 = int(eng.sink_end[l // eng.Hkv])
        rows, acc = [], 0
        for b, sp in enumerate(tables[l]):
            if sp is None:
                continue
            lo, hi = sp
            i = per.get((l, b))
            fk = int(nk[i]) if i is not None else 0
            if i is not None:
                f0[i], mbase[i] = acc, lo - s0
            rows.append(BlockRow(lo, hi, acc, fk))
            acc += fk
        led.blocks[l] = rows
        eng.splits[l] = 0
    if probs:
        _write_fine(eng, km, f0, mbase)
    _refresh_counts(eng, range(eng.L))
    if cfg.hierarchy is not None:
        _hierarchy(eng, [(l, b, block_seed(cfg.seed, _head(eng, l), b, 1)) for l in range(eng.L)
                         for b in range(len(led.blocks[l]))])


# ---------------------------------------------------------------------------- hierarchy


def _hierarchy(eng, jobs) -> None:
    """Coarse level of the given (ledger, block, seed) jobs (clustering.py:210-264).  Jobs of
    one ledger must be its LAST blocks in ascending order (coarse clusters are laid out in
    block order, so rebuilding the tail keeps every earlier block's coarse ids)."""
    cfg, led = eng.cfg, eng.led
    probs, inits, meta = [], [], []
    for (l, b, seed) in jobs:
        r = led.blocks[l][b]
        if r.fk == 0:
            meta.append(None)
            continue
        k1 = min(r.fk, max(1, -(-(r.end - r.start) // cfg.hierarchy.r1)))
        pick = np.random.default_rng(seed).choice(r.fk, size=k1, replace=False)
        probs.append((l, r.f0, r.fk, k1))
        inits.append(led.kc64[l, r.f0 + torch.as_tensor(pick, device=eng.device)])
        meta.append(len(probs) - 1)
    nk = np.zeros(0, np.int64)
    km = None
    if probs:
        km = KMeansBatch(eng.device, eng.d, probs, torch.cat(inits), pts64=led.kc64, wts=led.size,
                         rows64_cap=led.kcap, min_iters=cfg.refine_kmeans_iters)
        km.lloyd()
        nk = km.nonempty()
    c0 = np.zeros(len(probs), np.int64)
    mbase = np.zeros(len(probs), np.int64)
    for (l, b, _), pi in zip(jobs, meta):
        rows = led.blocks[l]
        start = rows[b - 1].c0 + rows[b - 1].ck if b > 0 else 0
        rows[b].c0 = start
        rows[b].ck = int(nk[pi]) if pi is not None else 0
        if pi is not None:
            c0[pi], mbase[pi] = start, rows[b].f0
    if probs:
        _write_coarse(eng, km, c0, mbase)
    _refresh_counts(eng, sorted({j[0] for j in jobs}))


# ---------------------------------------------------------------------------- online update


class _Ticks:
    """MPA_UPD_TRACE=1: device-synchronised wall time per phase of an online update (stderr)."""

    def __init__(self):
        import os
        import time

        self.on = os.environ.get("MPA_UPD_TRACE") in ("1", "2")
        self.sync = os.environ.get("MPA_UPD_TRACE") == "1"  # "2": host time only (no syncs)
        self.t = time.perf_counter
        self.last = self.t() if self.on else 0.0
        self.parts = []

    def __call__(self, name):
        if self.on:
            if self.sync:
                torch.cuda.synchronize()
            now = self.t()
            self.parts.append((name, (now - self.last) * 1e3))
            self.last = now

    def dump(self):
        if self.on:
            import sys

            ms = torch.cuda.memory_stats()
            print("update phases ms: " + ", ".join(f"{n} {v:.2f}" for n, v in self.parts)
                  + f" | segments {ms.get('segment.all.allocated', 0)} retries {ms.get('num_alloc_retries', 0)}",
                  file=sys.stderr)


def online_update(eng, seqs, cursor: int, samples: np.ndarray | None = None) -> dict:
    """Absorb the oldest L buffered tokens of every kv-head of `seqs` into the final block
    (clustering.py:404-472), then split / settle (:359-401) and refresh the final block's
    hierarchy (:465-471).  Returns timing-free counters (rounds, splits)."""
    cfg, led = eng.cfg, eng.led
    tick = _Ticks()
    L = cfg.local_buffer
    n_new = -(-L // cfg.fine_ratio)
    ledgers = [s * eng.Hkv + h for s in seqs for h in range(eng.Hkv)]
    for s in seqs:
        if eng.cache_len[s] - eng.buffer_start[s] < 2 * L:
            raise RuntimeError(f"buffer underflow: have {eng.cache_len[s] - eng.buffer_start[s]} tokens, need {2 * L}")
    # per-ledger problem layout, vectorised over the ledgers (clustering.py:430-434): problem
    # centroids = the final block's clusters, then the sampled buffer tokens
    Ls = np.asarray(ledgers, np.int64)
    S = Ls // eng.Hkv
    fin = [led.blocks[l][-1] for l in ledgers]
    F0 = np.fromiter((r.f0 for r in fin), np.int64, len(fin))
    FK = np.fromiter((r.fk for r in fin), np.int64, len(fin))
    FS = np.fromiter((r.start for r in fin), np.int64, len(fin))
    BS = eng.buffer_start[S].astype(np.int64)
    # the draw depends on (seed, cursor, kv-head) only (pipeline.py:170-172): once per head
    if samples is not None:  # drawn by the caller's generator (module-level append_tokens)
        samp_tab = np.broadcast_to(np.asarray(samples, np.int64).reshape(1, n_new), (eng.Hkv, n_new))
    else:
        samp_tab = np.stack([update_rng(cfg.seed, cursor, h).choice(L, size=n_new, replace=False)
                             for h in range(eng.Hkv)]).astype(np.int64)
    SAMP = samp_tab[Ls % eng.Hkv]                                    # [n, n_new]
    base = np.concatenate([[0], np.cumsum(FK + n_new)[:-1]]).astype(np.int64)
    c_at = int((FK + n_new).sum())
    probs = list(zip(Ls.tolist(), FS.tolist(), (BS + L - FS).tolist(), (FK + n_new).tolist()))
    tails = (BS - FS).tolist()
    dev = eng.device
    tick("loop")
    # gather indices built on the device from the per-ledger table (one small copy):
    # old centroid rows (ledger, f0 + i) -> (base + i), sampled buffer tokens -> (base + fk + s)
    n_l, no = len(ledgers), int(FK.sum())
    tab = torch.as_tensor(np.concatenate([Ls * led.kcap + F0, base, FK, Ls * eng.tcap + BS, SAMP.ravel()]),
                          dtype=torch.int64).to(dev, non_blocking=True)
    src0, base_d, fk_d, nsrc0 = tab[:n_l], tab[n_l:2 * n_l], tab[2 * n_l:3 * n_l], tab[3 * n_l:4 * n_l]
    of = torch.repeat_interleave(torch.arange(n_l, device=dev), fk_d, output_size=no)
    intra = torch.arange(no, device=dev) - (torch.cumsum(fk_d, 0) - fk_d)[of]
    osrc, odst = src0[of] + intra, base_d[of] + intra
    nsrc = (nsrc0[:, None] + tab[4 * n_l:].view(n_l, n_new)).view(-1)
    ndst = ((base_d + fk_d)[:, None] + torch.arange(n_new, device=dev)).view(-1)
    tick("idx")
    cache = eng.__dict__.setdefault("_upd_scratch", {})
    init = _scratch(cache, "init", c_at * eng.d, torch.float64, dev).view(c_at, eng.d)
    # through a kept scratch block: a fresh ~30 MB temporary every event (its size creeps up)
    # sends the caching allocator to cudaMalloc, which stalls for tens of ms at times
    g = _scratch(cache, "gather", no * eng.d, torch.float64, dev).view(no, eng.d)
    torch.index_select(led.kc64.view(-1, eng.d), 0, osrc, out=g)
    init.index_copy_(0, odst, g)
    tick("init_old")
    init[ndst] = eng.k_raw.view(-1, eng.d)[nsrc].double()
    tick("init_new")
    counts = torch.zeros(c_at, dtype=torch.int32, device=dev)
    counts[odst] = led.size.view(-1)[osrc]
    tick("counts0")
    km = KMeansBatch(dev, eng.d, probs, init, pts=eng.k_raw, tcap=eng.tcap,
                     min_iters=cfg.refine_kmeans_iters, count_init=counts, cache=cache)
    dist = _scratch(cache, "dist", len(probs) * L * km.k_max, torch.float64, dev).view(len(probs), L, km.k_max)
    tails_d = _i32(eng, tails)
    tick("batch")
    call("mpa_km_seq_assign", km.struct(), ptr(tails_d), L, ptr(dist), stream_ptr())
    tick("seq_assign")
    mbase = FS - eng.sink_end[S].astype(np.int64)
    rounds = km.lloyd()
    tick(f"lloyd({rounds})")
    nk = km.nonempty()
    tick("nonempty")
    _write_fine(eng, km, F0, mbase)  # queued before the host bookkeeping below
    for i, l in enumerate(ledgers):
        F = led.blocks[l][-1]
        F.end = int(eng.buffer_start[l // eng.Hkv]) + L
        F.fk = int(nk[i])
    tick("write")
    for s in seqs:
        eng.buffer_start[s] += L
    eng._sync_scalars()
    _refresh_counts(eng, ledgers)
    tick("counts")
    n_splits = _split(eng, ledgers)
    tick("split")
    if cfg.hierarchy is not None:
        _hierarchy(eng, [(l, len(led.blocks[l]) - 1,
                          block_seed(cfg.seed, _head(eng, l), int(eng.buffer_start[l // eng.Hkv]), 3))
                         for l in ledgers])
        tick("hierarchy")
    tick.dump()
    return {"rounds": rounds, "splits": n_splits}


def _split(eng, ledgers, settle: bool = True) -> int:
    """Seal the first W tokens of every final block with |final| >= W + alpha; both sides are
    seeded with their members' means and (settle=True) settled with Lloyd(min_iters=0)."""
    cfg, led = eng.cfg, eng.led
    W, A = cfg.block_size, cfg.alpha
    total = 0
    while True:
        todo = [l for l in ledgers if led.blocks[l][-1].end - led.blocks[l][-1].start >= W + A]
        if not todo:
            return total
        total += len(todo)
        # (1) side means from the current membership
        probs, firsts, ncl = [], [], []
        for l in todo:
            F = led.blocks[l][-1]
            cut = F.start + W
            probs += [(l, F.start, W, F.fk), (l, cut, F.end - cut, F.fk)]
            firsts += [F.f0, F.f0]
            ncl += [F.fk, F.fk]
        dev = eng.device
        km = KMeansBatch(dev, eng.d, probs, torch.zeros(sum(p[3] for p in probs), eng.d, dtype=torch.float64,
                                                         device=dev), pts=eng.k_raw, tcap=eng.tcap)
        firsts_d, ncl_d = _i32(eng, firsts), _i32(eng, ncl)
        call("mpa_km_assign_from_level", km.struct(), ptr(led.off), ptr(led.mem), led.kcap, led.tcap, ptr(firsts_d),
             ptr(ncl_d), None, stream_ptr())
        km.means()
        if settle:
            # (2) settle each side from its non-empty side means (clustering.py:384-394)
            sprobs, sinit = [], []
            for i, (l, lo, n, k) in enumerate(probs):
                live = km.counts(i) > 0
                c = km.centroids(i)[live]
                sprobs.append((l, lo, n, int(c.shape[0])))
                sinit.append(c)
            st = KMeansBatch(dev, eng.d, sprobs, torch.cat(sinit), pts=eng.k_raw, tcap=eng.tcap, min_iters=0)
            st.lloyd()
        else:
            # positional pages: straddlers split, no settle (clustering.py:540); the side problems
            # are written as they are (empty sides dropped by the compaction, clustering.py:377)
            st, sprobs = km, probs
        nk = st.nonempty()
        f0 = np.zeros(len(sprobs), np.int64)
        mbase = np.zeros(len(sprobs), np.int64)
        for j, l in enumerate(todo):
            s0 = int(eng.sink_end[l // eng.Hkv])
            F = led.blocks[l][-1]
            cut = F.start + W
            left = BlockRow(F.start, cut, F.f0, int(nk[2 * j]), F.c0, 0)
            right = BlockRow(cut, F.end, F.f0 + int(nk[2 * j]), int(nk[2 * j + 1]), F.c0, 0)
            f0[2 * j], mbase[2 * j] = left.f0, left.start - s0
            f0[2 * j + 1], mbase[2 * j + 1] = right.f0, right.start - s0
            led.blocks[l][-1:] = [left, right]
            eng.splits[l] += 1
        _write_fine(eng, st, f0, mbase)
        _refresh_counts(eng, todo)
        if cfg.hierarchy is not None:
            _hierarchy(eng, [(l, len(led.blocks[l]) - 2, block_seed(cfg.seed, _head(eng, l), len(led.blocks[l]) - 2, 2))
                             for l in todo])


# ---------------------------------------------------------------------------- positional pages


def _page_batch(eng, spans):
    """KMeansBatch whose assignment is the contiguous r-token page of each point, with means."""
    r = eng.cfg.fine_ratio
    probs = [(l, lo, hi - lo, -(-(hi - lo) // r)) for (l, lo, hi) in spans]
    km = KMeansBatch(eng.device, eng.d, probs, torch.zeros(sum(p[3] for p in probs), eng.d, dtype=torch.float64,
                                                          device=eng.device), pts=eng.k_raw, tcap=eng.tcap)
    asg = [torch.arange(p[2], device=eng.device, dtype=torch.int32) // r for p in probs]
    if asg:
        flat = torch.cat(asg)
        km.assign[: flat.numel()].copy_(flat)
        km.means()
    return km


def prefill_positional(eng) -> None:
    """Positional comparator: contiguous r-token pages with mean centroids (clustering.py:497-526)."""
    cfg, led = eng.cfg, eng.led
    W = cfg.block_size
    eng.set_prompt_layout()
    spans, owners = [], []
    for l in range(eng.L):
        s = l // eng.Hkv
        s0, b0 = int(eng.sink_end[s]), int(eng.buffer_start[s])
        nsealed = (b0 - s0) // W
        rows = []
        for b in range(nsealed + 1):
            lo = s0 + b * W
            hi = lo + W if b < nsealed else b0
            rows.append(BlockRow(lo, hi, 0, 0))
            if hi > lo:
                spans.append((l, lo, hi))
                owners.append((l, b))
        led.blocks[l] = rows
    km = _page_batch(eng, spans)
    nk = km.nonempty()
    f0 = np.zeros(len(spans), np.int64)
    mbase = np.zeros(len(spans), np.int64)
    per = {o: i for i, o in enumerate(owners)}
    for l in range(eng.L):
        acc = 0
        s0 = int(eng.sink_end[l // eng.Hkv])
        for b, row in enumerate(led.blocks[l]):
            row.f0 = acc
            i = per.get((l, b))
            if i is not None:
                row.fk = int(nk[i])
                f0[i], mbase[i] = acc, row.start - s0
            acc += row.fk
    if spans:
        _write_fine(eng, km, f0, mbase)
    _refresh_counts(eng, range(eng.L))


def positional_update(eng, seqs) -> dict:
    """Rebuild the final block's pages over the absorbed tokens, then split without settling
    (clustering.py:529-541)."""
    cfg, led = eng.cfg, eng.led
    L = cfg.local_buffer
    ledgers = [s * eng.Hkv + h for s in seqs for h in range(eng.Hkv)]
    spans = []
    for l in ledgers:
        s = l // eng.Hkv
        if eng.cache_len[s] - eng.buffer_start[s] < 2 * L:
            raise RuntimeError("buffer underflow")
        F = led.blocks[l][-1]
        spans.append((l, F.start, int(eng.buffer_start[s]) + L))
    km = _page_batch(eng, spans)
    nk = km.nonempty()
    f0 = np.zeros(len(spans), np.int64)
    mbase = np.zeros(len(spans), np.int64)
    for i, l in enumerate(ledgers):
        F = led.blocks[l][-1]
        f0[i], mbase[i] = F.f0, F.start - int(eng.sink_end[l // eng.Hkv])
        F.end, F.fk = spans[i][2], int(nk[i])
    _write_fine(eng, km, f0, mbase)
    for s in seqs:
        eng.buffer_start[s] += L
    eng._sync_scalars()
    _refresh_counts(eng, ledgers)
    return {"rounds": 0, "splits": _split(eng, ledgers, settle=False)}


# ============================================================================ reference API
# The module-level surface of pkg/src/multipole_attn/clustering.py (same names, arguments, return
# types and exceptions) for callers holding numpy arrays.  k-means runs on the batched Lloyd kernels
# (fp64 points); block indices, updates and the positional comparator run on a one-ledger engine
# (the serving code path, fp32 cache); means, nearest-centroid checks and squared errors run on the
# fp64 kernels of csrc/mpa_refapi.cu.  Only bookkeeping over the returned arrays stays on the host.

import hashlib as _hashlib
import json as _json
from dataclasses import dataclass as _dataclass

MAX_EXTRA_ITERS = 100  # clustering.py:30 (csrc/mpa_cluster.cu kMaxExtraRounds)


class LedgerAuditError(AssertionError):
    """clustering.py:33."""


@_dataclass
class Cluster:
    """clustering.py:37-43."""

    key_centroid: np.ndarray
    value_centroid: np.ndarray | None
    size: int
    member_indices: np.ndarray
    children: list | None = None


@_dataclass
class Block:
    """clustering.py:46-54."""

    start: int
    end: int
    clusters: list
    level1: list | None = None

    def __len__(self) -> int:
        return self.end - self.start


@_dataclass
class BlockLedger:
    """clustering.py:57-77."""

    sink_end: int
    sealed: list
    final: Block
    buffer_start: int
    total: int
    split_count: int = 0

    @property
    def buffer_len(self) -> int:
        return self.total - self.buffer_start

    def blocks(self) -> list:
        return self.sealed + [self.final]

    def clustered_tokens(self) -> int:
        return self.buffer_start - self.sink_end


def _device():
    from . import _dev

    return _dev.device()


def lloyd(points, init_centroids, min_iters: int):
    """clustering.py:123-143 on the batched Lloyd kernels (fp64 points, no weights): rounds until an
    assignment pass is a fixed point after >= min_iters updates; (centroids, assignment)."""
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    init = np.array(init_centroids, dtype=np.float64)
    n, d = pts.shape
    k = init.shape[0]
    dev = _device()
    km = KMeansBatch(dev, d, [(0, 0, n, k)], torch.as_tensor(init, device=dev),
                     pts64=torch.as_tensor(pts, device=dev), rows64_cap=n, min_iters=min_iters)
    km.lloyd()
    return km.cent.cpu().numpy(), km.assign[:n].cpu().numpy().astype(np.int64)


def _clusters_from_assignment(points, centroids, assign, base_index, index_map=None):
    """clustering.py:146-167: empty clusters dropped, ids compacted in centroid order."""
    out = []
    for cid in range(centroids.shape[0]):
        local = np.flatnonzero(assign == cid)
        if local.size == 0:
            continue
        idx = np.sort(index_map[local]) if index_map is not None else local.astype(np.int64) + base_index
        out.append(Cluster(key_centroid=centroids[cid].copy(), value_centroid=None, size=int(local.size),
                           member_indices=idx))
    return out


def kmeans(points, k: int, iters: int, seed: int) -> list:
    """clustering.py:170-184: random-point init (host PCG64, the reference's draw), device Lloyd."""
    points = np.asarray(points, dtype=np.float64)
    n = points.shape[0]
    if n == 0:
        raise ValueError("points must be nonempty")
    if k < 1:
        raise ValueError("k must be >= 1")
    k = min(k, n)
    init = points[np.random.default_rng(seed).choice(n, size=k, replace=False)]
    centroids, assign = lloyd(points, init, iters)
    return _clusters_from_assignment(points, centroids, assign, base_index=0)


def fill_value_centroids(clusters: list, values) -> None:
    """clustering.py:187-192: value centroid = in-order mean of the members' values (device)."""
    from . import _dev

    if not clusters:
        return
    vals = np.asarray(values, dtype=np.float64)
    mean, _ = _dev.seg_stats(vals, [c.member_indices for c in clusters])
    for c, v in zip(clusters, mean):
        c.value_centroid = v


def wcss(ledger: BlockLedger, keys) -> float:
    """clustering.py:195-203: within-cluster sum of squared distances over all fine clusters."""
    from . import _dev

    clusters = [c for b in ledger.blocks() for c in b.clusters]
    if not clusters:
        return 0.0
    _, sq = _dev.seg_stats(np.asarray(keys, dtype=np.float64), [c.member_indices for c in clusters],
                           centroids=np.stack([c.key_centroid for c in clusters]))
    return sq


def build_hierarchy(clusters: list, cfg, block_len: int, seed: int) -> list:
    """clustering.py:210-264: size-weighted Lloyd over the fine key centroids on the device; coarse
    key / value centroids are the size-weighted means of their children (exact member means)."""
    from . import _dev

    if cfg.hierarchy is None:
        raise ConfigError("hierarchy is not enabled")
    if not clusters:
        return []
    fine_kc = np.ascontiguousarray(np.stack([c.key_centroid for c in clusters]))
    weights = np.array([c.size for c in clusters], dtype=np.float64)
    k1 = min(len(clusters), max(1, -(-block_len // cfg.hierarchy.r1)))
    init = fine_kc[np.random.default_rng(seed).choice(len(clusters), size=k1, replace=False)].copy()
    n, d = fine_kc.shape
    dev = _device()
    km = KMeansBatch(dev, d, [(0, 0, n, k1)], torch.as_tensor(init, device=dev),
                     pts64=torch.as_tensor(fine_kc, device=dev),
                     wts=torch.as_tensor(weights.astype(np.int32), device=dev), rows64_cap=n,
                     min_iters=cfg.refine_kmeans_iters)
    km.lloyd()
    assign = km.assign[:n].cpu().numpy()
    groups = [np.flatnonzero(assign == cid) for cid in range(k1)]
    groups = [g for g in groups if g.size]
    kc, _ = _dev.seg_stats(fine_kc, groups, weights=weights)
    vc, _ = _dev.seg_stats(np.stack([c.value_centroid for c in clusters]), groups, weights=weights)
    out = []
    for j, g in enumerate(groups):
        members = [clusters[i] for i in g]
        out.append(Cluster(key_centroid=kc[j], value_centroid=vc[j], size=int(sum(c.size for c in members)),
                           member_indices=np.sort(np.concatenate([c.member_indices for c in members])),
                           children=[int(i) for i in g]))
    return out


def _one_ledger_engine(keys, values, n_tok: int, cfg, head: int, mode: str = "multipole", tcap: int | None = None):
    from .core import HeadLayout
    from .engine import DecodeEngine

    keys = np.asarray(keys, dtype=np.float32)
    values = np.asarray(values, dtype=np.float32)
    d = keys.shape[-1]
    eng = DecodeEngine(cfg, HeadLayout(1, 1, d), 1, tcap=max(16, tcap or n_tok + 1), dtype=torch.float32, mode=mode)
    eng.head_ids = np.array([head])
    dev = eng.device
    eng.write_tokens(torch.as_tensor(keys[None, None, :n_tok], device=dev),
                     torch.as_tensor(values[None, None, :n_tok], device=dev))
    return eng


def _to_block_ledger(eng, l: int = 0) -> BlockLedger:
    """The engine's ledger l as reference objects (Cluster lists per block, coarse level1)."""
    h = eng.export_ledger(l)
    off = np.zeros(h.size.size + 1, np.int64)
    np.cumsum(h.size, out=off[1:])
    blocks = []
    for r in h.blocks:
        cl = [Cluster(key_centroid=h.kc[i].copy(), value_centroid=h.vc[i].copy(), size=int(h.size[i]),
                      member_indices=np.sort(h.mem[off[i]:off[i + 1]]).astype(np.int64))
              for i in range(r.f0, r.f0 + r.fk)]
        lvl = None
        if h.csize is not None:
            lvl = []
            for j in range(r.c0, r.c0 + r.ck):
                kids = [int(c) - r.f0 for c in h.child[h.child_off[j]:h.child_off[j + 1]]]
                lvl.append(Cluster(key_centroid=h.ckc[j].copy(), value_centroid=h.cvc[j].copy(),
                                   size=int(h.csize[j]),
                                   member_indices=np.sort(np.concatenate([cl[c].member_indices for c in kids])),
                                   children=kids))
        blocks.append(Block(r.start, r.end, cl, lvl))
    return BlockLedger(sink_end=h.sink_end, sealed=blocks[:-1], final=blocks[-1], buffer_start=h.buffer_start,
                       total=h.total, split_count=h.splits)


def _to_host_ledger(ledger: BlockLedger, hier: bool):
    from .ledger import BlockRow, HostLedger

    rows, kcs, vcs, sizes, mem = [], [], [], [], []
    ckc, cvc, csz, child, coff = [], [], [], [], [0]
    f0 = c0 = 0
    for b in ledger.blocks():
        ck = len(b.level1) if (hier and b.level1 is not None) else 0
        rows.append(BlockRow(b.start, b.end, f0, len(b.clusters), c0, ck))
        for c in b.clusters:
            kcs.append(c.key_centroid)
            vcs.append(c.value_centroid)
            sizes.append(c.size)
            mem.append(np.asarray(c.member_indices, np.int64))
        if ck:
            for c in b.level1:
                ckc.append(c.key_centroid)
                cvc.append(c.value_centroid)
                csz.append(c.size)
                child.extend(f0 + int(x) for x in c.children)
                coff.append(len(child))
        f0 += len(b.clusters)
        c0 += ck
    d = len(kcs[0]) if kcs else 1
    h = HostLedger(ledger.sink_end, ledger.buffer_start, ledger.total, ledger.split_count, rows,
                   np.stack(kcs) if kcs else np.zeros((0, d)), np.stack(vcs) if vcs else np.zeros((0, d)),
                   np.array(sizes, np.int64), np.concatenate(mem) if mem else np.zeros(0, np.int64))
    if hier:
        h.ckc = np.stack(ckc) if ckc else np.zeros((0, d))
        h.cvc = np.stack(cvc) if cvc else np.zeros((0, d))
        h.csize = np.array(csz, np.int64)
        h.child_off = np.array(coff, np.int64)
        h.child = np.array(child, np.int64)
    return h


def build_prefill_index_head(keys, values, prompt_len: int, cfg, head: int) -> BlockLedger:
    """clustering.py:288-326: blockwise clustering of one head's prompt on the engine's kernels."""
    if prompt_len <= cfg.sink_tokens:
        raise ConfigError(f"prompt_len {prompt_len} must exceed sink_tokens {cfg.sink_tokens}")
    eng = _one_ledger_engine(keys, values, prompt_len, cfg, head)
    eng.prefill()
    return _to_block_ledger(eng)


def build_prefill_index(trace, cfg) -> list:
    """clustering.py:329-340: one ledger per kv-head over the trace's prompt."""
    return [build_prefill_index_head(trace.keys[h, : trace.prompt_len], trace.values[h, : trace.prompt_len],
                                     trace.prompt_len, cfg, h) for h in range(trace.layout.num_kv_heads)]


def _reload(ledger: BlockLedger, keys, values, cfg, head: int, mode: str):
    eng = _one_ledger_engine(keys, values, ledger.total, cfg, head, mode=mode,
                             tcap=max(ledger.total + 1, np.asarray(keys).shape[0] + 1))
    eng.load_ledgers([_to_host_ledger(ledger, cfg.hierarchy is not None)])
    return eng


def _replace(dst: BlockLedger, src: BlockLedger) -> BlockLedger:
    dst.sink_end, dst.sealed, dst.final = src.sink_end, src.sealed, src.final
    dst.buffer_start, dst.total, dst.split_count = src.buffer_start, src.total, src.split_count
    return dst


def append_tokens(ledger: BlockLedger, keys, values, cfg, rng: np.random.Generator, head: int = 0) -> BlockLedger:
    """clustering.py:404-472: absorb the oldest L buffered tokens into the final block (sampled
    centroids drawn from `rng` like the reference, sequential running-mean assignment, Lloyd
    refinement, split / settle, hierarchy refresh) on the engine's update kernels.  Mutates and
    returns the ledger."""
    L = cfg.local_buffer
    if ledger.buffer_len < 2 * L:
        raise RuntimeError(f"buffer underflow: have {ledger.buffer_len} tokens, need {2 * L}")
    n_new = -(-L // cfg.fine_ratio)
    sampled = rng.choice(L, size=n_new, replace=False)
    eng = _reload(ledger, keys, values, cfg, head, "multipole")
    online_update(eng, [0], 0, samples=sampled)
    return _replace(ledger, _to_block_ledger(eng))


def build_positional_index_head(keys, values, prompt_len: int, cfg) -> BlockLedger:
    """clustering.py:497-526: contiguous pages of r tokens with page-mean centroids."""
    if prompt_len <= cfg.sink_tokens:
        raise ConfigError(f"prompt_len {prompt_len} must exceed sink_tokens {cfg.sink_tokens}")
    eng = _one_ledger_engine(keys, values, prompt_len, cfg, 0, mode="positional-baseline")
    eng.prefill()
    return _to_block_ledger(eng)


def append_tokens_positional(ledger: BlockLedger, keys, values, cfg) -> BlockLedger:
    """clustering.py:529-541: positional-page analogue of append_tokens."""
    L = cfg.local_buffer
    if ledger.buffer_len < 2 * L:
        raise RuntimeError("buffer underflow")
    eng = _reload(ledger, keys, values, cfg, 0, "positional-baseline")
    positional_update(eng, [0])
    return _replace(ledger, _to_block_ledger(eng))


def audit_ledger(ledger: BlockLedger, keys, cfg, values=None, rel_tol: float = 1e-5,
                 check_assignment: bool = True) -> None:
    """clustering.py:548-623: raise LedgerAuditError on a violated invariant (partition, spans,
    final-block size, centroid = member mean, nearest assignment).  Index bookkeeping on the host,
    the numeric checks on the device."""
    from . import _dev

    keys64 = np.asarray(keys, dtype=np.float64)
    pieces = [np.arange(0, ledger.sink_end, dtype=np.int64)]
    for block in ledger.blocks():
        for c in block.clusters:
            pieces.append(np.asarray(c.member_indices, np.int64))
            if c.size != len(c.member_indices):
                raise LedgerAuditError("cluster size disagrees with member count")
    pieces.append(np.arange(ledger.buffer_start, ledger.total, dtype=np.int64))
    flat = np.sort(np.concatenate(pieces))
    if flat.size != ledger.total or not np.array_equal(flat, np.arange(ledger.total, dtype=np.int64)):
        raise LedgerAuditError("token indices do not tile [0, total) exactly")
    cursor = ledger.sink_end
    for block in ledger.sealed:
        if block.start != cursor or len(block) != cfg.block_size:
            raise LedgerAuditError("sealed block spans are not contiguous W-sized")
        cursor = block.end
    if ledger.final.start != cursor or ledger.final.end != ledger.buffer_start:
        raise LedgerAuditError("final block span inconsistent with buffer start")
    if len(ledger.final) > cfg.block_size + cfg.alpha:
        raise LedgerAuditError("final block exceeds W + alpha")
    if ledger.split_count > 0 and len(ledger.final) < cfg.alpha:
        raise LedgerAuditError("final block shorter than alpha after a split")
    values64 = None if values is None else np.asarray(values, dtype=np.float64)
    for block in ledger.blocks():
        if not block.clusters:
            continue
        members = [np.asarray(c.member_indices, np.int64) for c in block.clusters]
        idx = np.concatenate(members)
        if idx.size and (idx.min() < block.start or idx.max() >= block.end):
            raise LedgerAuditError("cluster member outside its block span")
        centroids = np.stack([c.key_centroid for c in block.clusters])
        means, _ = _dev.seg_stats(keys64, members)
        scale = max(1.0, float(np.max(np.abs(centroids))))
        if np.max(np.abs(means - centroids)) > rel_tol * scale:
            raise LedgerAuditError("key centroid drifted from member mean")
        if values64 is not None:
            vcent = np.stack([c.value_centroid for c in block.clusters])
            vmeans, _ = _dev.seg_stats(values64, members)
            vscale = max(1.0, float(np.max(np.abs(vcent))))
            if np.max(np.abs(vmeans - vcent)) > rel_tol * vscale:
                raise LedgerAuditError("value centroid drifted from member mean")
        if check_assignment:
            owner = np.concatenate([np.full(c.size, cid) for cid, c in enumerate(block.clusters)])
            if not np.array_equal(_dev.nearest(keys64[idx], centroids), owner):
                raise LedgerAuditError("a member is not assigned to its nearest centroid")


def ledger_diagnostic(ledger: BlockLedger) -> dict:
    """clustering.py:626-650: JSON-friendly summary (spans, sizes, centroid checksums)."""

    def checksum(arr) -> str:
        return _hashlib.sha256(np.ascontiguousarray(arr, dtype="<f8").tobytes()).hexdigest()[:16]

    def block_doc(block: Block) -> dict:
        doc = {"span": [block.start, block.end], "cluster_sizes": [c.size for c in block.clusters],
               "key_centroid_checksums": [checksum(c.key_centroid) for c in block.clusters]}
        if block.level1 is not None:
            doc["level1_sizes"] = [c.size for c in block.level1]
        return doc

    return {"sink_end": ledger.sink_end, "buffer": [ledger.buffer_start, ledger.total],
            "split_count": ledger.split_count, "sealed": [block_doc(b) for b in ledger.sealed],
            "final": block_doc(ledger.final)}


def dump_ledger_json(ledger: BlockLedger) -> str:
    """clustering.py:653-654."""
    return _json.dumps(ledger_diagnostic(ledger), sort_keys=True)


def load_ledger_json(doc: str) -> dict:
    """clustering.py:657."""
    return _json.loads(doc)
