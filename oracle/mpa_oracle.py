"""CPU ORACLE for the Multipole Attention decode path -- TEST INFRASTRUCTURE ONLY.

This is a numpy restatement of the reference package `multipole_attn`
(/root/reference/pkg/src/multipole_attn/*.py).  It is the *checker* for the CUDA
product path; it is never the thing measured or shipped.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and the
`--impl reference` arm) may import it.

Parity is PINNED: `tests/golden/make_golden.py` runs the real reference (imported
from /root/reference in the build container) on seeded inputs and commits the
results under `tests/golden/*.npz`; `tests/test_golden_oracle.py` checks that this
restatement reproduces them bit-for-bit (selections, ledgers, fp64 outputs).

Every floating-point primitive whose rounding can decide a discrete outcome
(argmin / argmax / sort order) uses the same numpy call as the reference:
einsum for squared norms, BLAS `@` for contractions, `np.add.at` / `np.mean`
(sequential in member order) for means, `np.exp` for scores.

Data model: instead of the reference's Cluster objects the oracle keeps one
`Level` per (block, level) holding stacked centroids and member lists, which is
also the shape the device ledger (paper_2506_13059_b200/ledger.py) converts to.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from paper_2506_13059_b200.core import (
    ConfigError,
    EngineConfig,
    HeadLayout,
    KvTrace,
    block_seed,
    inv_freq,
    update_rng,
)

EXTRA_LLOYD_ROUNDS = 100  # clustering.py:30 MAX_EXTRA_ITERS
MODES = ("multipole", "oracle", "flat-no-replacement", "positional-baseline")  # pipeline.py:23


# ---------------------------------------------------------------------------
# Rotary views (rope.py:37-68)


def rotate(v, pos, head_dim: int, theta: float) -> np.ndarray:
    """Interleaved-pair rotation (2i, 2i+1) by pos*theta^(-2i/d), fp64 (rope.py:37-53)."""
    v = np.asarray(v, dtype=np.float64)
    ang = np.multiply.outer(np.asarray(pos, dtype=np.float64), inv_freq(head_dim, theta))
    cs, sn = np.cos(ang), np.sin(ang)
    ev, od = v[..., 0::2], v[..., 1::2]
    out = np.empty_like(v)
    out[..., 0::2] = ev * cs - od * sn
    out[..., 1::2] = ev * sn + od * cs
    return out


def lookup_query(q, cfg: EngineConfig, d: int) -> np.ndarray:
    """Query rotated at the fixed window offset Delta (rope.py:66-68)."""
    return rotate(q, cfg.window_offset, d, cfg.rope_theta)


# ---------------------------------------------------------------------------
# Ledger data model


@dataclass
class Level:
    """Clusters of one block at one level (fine = 2, coarse = 1)."""

    kc: np.ndarray                      # (k, d) fp64 key centroids (raw-key view)
    vc: np.ndarray | None               # (k, d) fp64 value centroids
    members: list                       # k sorted int64 arrays of global token ids
    children: list | None = None        # coarse only: fine ids (ascending) per cluster

    @property
    def k(self) -> int:
        return len(self.members)

    @property
    def sizes(self) -> np.ndarray:
        return np.array([m.size for m in self.members], dtype=np.int64)


@dataclass
class BlockO:
    start: int
    end: int
    fine: Level
    coarse: Level | None = None


@dataclass
class LedgerO:
    sink_end: int
    blocks: list                        # sealed blocks..., final block last
    buffer_start: int
    total: int
    splits: int = 0

    @property
    def final(self) -> BlockO:
        return self.blocks[-1]

    @property
    def buffer_len(self) -> int:
        return self.total - self.buffer_start


def empty_level(d: int) -> Level:
    return Level(np.zeros((0, d)), np.zeros((0, d)), [])


# ---------------------------------------------------------------------------
# Lloyd's algorithm (clustering.py:84-184)


def sq_dists(p: np.ndarray, c: np.ndarray) -> np.ndarray:
    """||p||^2 + ||c||^2 - 2 p.c, fp64, (n, k) (clustering.py:84-88)."""
    pn = np.einsum("nd,nd->n", p, p)
    cn = np.einsum("kd,kd->k", c, c)
    return pn[:, None] + cn[None, :] - 2.0 * p @ c.T


def assign_nearest(p: np.ndarray, c: np.ndarray) -> np.ndarray:
    """First-minimum argmin over sq_dists (clustering.py:134)."""
    return np.argmin(sq_dists(p, c), axis=1)


def assign_margin(p: np.ndarray, c: np.ndarray) -> np.ndarray:
    """(second best - best) / max(|best|, 1) per row: rows below ~1e-12 are true ties."""
    dist = sq_dists(p, c)
    if dist.shape[1] < 2:
        return np.full(dist.shape[0], np.inf)
    part = np.partition(dist, 1, axis=1)
    return (part[:, 1] - part[:, 0]) / np.maximum(np.abs(part[:, 0]), 1.0)


def repair_empty(p, c, lab) -> None:
    """Steal the farthest member of the largest cluster for each empty one, lowest empty id
    first; stop when none is empty or the largest has <= 1 member (clustering.py:91-110)."""
    k = c.shape[0]
    while True:
        cnt = np.bincount(lab, minlength=k)
        holes = np.flatnonzero(cnt == 0)
        if not holes.size:
            return
        donor = int(np.argmax(cnt))
        if cnt[donor] <= 1:
            return
        who = np.flatnonzero(lab == donor)
        diff = p[who] - c[donor]
        far = who[int(np.argmax(np.einsum("nd,nd->n", diff, diff)))]
        c[int(holes[0])] = p[far]
        lab[far] = int(holes[0])


def cluster_means(p, lab, k):
    """Sequential (np.add.at) member sums / counts; empty clusters stay 0 (clustering.py:113-120)."""
    acc = np.zeros((k, p.shape[1]))
    np.add.at(acc, lab, p)
    cnt = np.bincount(lab, minlength=k)
    res = acc.copy()
    live = cnt > 0
    res[live] /= cnt[live, None]
    return res, cnt


def lloyd(points, init, min_iters: int):
    """Assign/repair/update to a fixed point after >= min_iters updates (clustering.py:123-143)."""
    p = np.asarray(points, dtype=np.float64)
    c = np.array(init, dtype=np.float64)
    k = c.shape[0]
    last = None
    rounds = 0
    while True:
        lab = assign_nearest(p, c)
        repair_empty(p, c, lab)
        if last is not None and rounds >= min_iters and np.array_equal(lab, last):
            return c, lab
        if rounds >= min_iters + EXTRA_LLOYD_ROUNDS:
            return cluster_means(p, lab, k)[0], lab
        c = cluster_means(p, lab, k)[0]
        last = lab
        rounds += 1


def compact(c, lab, idmap: np.ndarray) -> Level:
    """Drop empty clusters, keep centroid order; members mapped through idmap (clustering.py:146-167)."""
    rows, mem = [], []
    for j in range(c.shape[0]):
        loc = np.flatnonzero(lab == j)
        if loc.size:
            rows.append(j)
            mem.append(np.sort(idmap[loc]).astype(np.int64))
    kc = c[rows].copy() if rows else np.zeros((0, c.shape[1]))
    return Level(kc, None, mem)


def kmeans(points, k: int, iters: int, seed: int, base: int = 0) -> Level:
    """Random-point init from default_rng(seed).choice(n, k, replace=False) (clustering.py:170-184)."""
    p = np.asarray(points, dtype=np.float64)
    n = p.shape[0]
    if n == 0:
        raise ValueError("points must be nonempty")
    if k < 1:
        raise ValueError("k must be >= 1")
    k = min(k, n)
    pick = np.random.default_rng(seed).choice(n, size=k, replace=False)
    c, lab = lloyd(p, p[pick], iters)
    return compact(c, lab, np.arange(n, dtype=np.int64) + base)


def value_means(level: Level, values) -> None:
    """Value centroid = np.mean over members, sequential (clustering.py:187-192)."""
    v64 = np.asarray(values, dtype=np.float64)
    d = v64.shape[1]
    level.vc = (np.stack([np.mean(v64[m], axis=0) for m in level.members])
                if level.members else np.zeros((0, d)))


# ---------------------------------------------------------------------------
# Hierarchy (clustering.py:210-264)


def coarse_level(fine: Level, cfg: EngineConfig, block_len: int, seed: int) -> Level:
    if cfg.hierarchy is None:
        raise ConfigError("hierarchy is not enabled")
    d = fine.kc.shape[1]
    if fine.k == 0:
        return Level(np.zeros((0, d)), np.zeros((0, d)), [], [])
    fk = fine.kc
    wt = fine.sizes.astype(np.float64)
    k1 = min(fine.k, max(1, -(-block_len // cfg.hierarchy.r1)))
    cen = fk[np.random.default_rng(seed).choice(fine.k, size=k1, replace=False)].copy()
    last, rounds = None, 0
    while True:
        lab = assign_nearest(fk, cen)
        repair_empty(fk, cen, lab)
        if last is not None and rounds >= cfg.refine_kmeans_iters and np.array_equal(lab, last):
            break
        if rounds >= cfg.refine_kmeans_iters + EXTRA_LLOYD_ROUNDS:
            break
        acc = np.zeros((k1, d))
        np.add.at(acc, lab, fk * wt[:, None])
        wsum = np.zeros(k1)
        np.add.at(wsum, lab, wt)
        live = wsum > 0
        cen[live] = acc[live] / wsum[live, None]
        last, rounds = lab, rounds + 1
    kcs, vcs, mem, kids = [], [], [], []
    for j in range(k1):
        ch = np.flatnonzero(lab == j)
        if not ch.size:
            continue
        n = sum(int(fine.members[i].size) for i in ch)
        # Python-level running sums starting from int 0, as the reference does.
        kcs.append(sum(fine.kc[i] * int(fine.members[i].size) for i in ch) / n)
        vcs.append(sum(fine.vc[i] * int(fine.members[i].size) for i in ch) / n)
        mem.append(np.sort(np.concatenate([fine.members[i] for i in ch])))
        kids.append([int(i) for i in ch])
    return Level(np.stack(kcs), np.stack(vcs), mem, kids)


# ---------------------------------------------------------------------------
# Prefill ledger + online update (clustering.py:272-472)


def _cluster_span(keys, values, lo, hi, cfg, seed) -> Level:
    d = np.asarray(keys).shape[1]
    if hi <= lo:
        return empty_level(d)
    pts = np.asarray(keys, dtype=np.float64)[lo:hi]
    lev = kmeans(pts, max(1, -(-(hi - lo) // cfg.fine_ratio)), cfg.prefill_kmeans_iters, seed, base=lo)
    value_means(lev, values)
    return lev


def prefill_ledger(keys, values, prompt_len: int, cfg: EngineConfig, head: int) -> LedgerO:
    """Sinks [0, S), floor(clustered/W) sealed W-blocks, final block, buffer of
    min(L, prompt - S) tokens (clustering.py:288-326)."""
    if prompt_len <= cfg.sink_tokens:
        raise ConfigError(f"prompt_len {prompt_len} must exceed sink_tokens {cfg.sink_tokens}")
    s0 = cfg.sink_tokens
    buf0 = prompt_len - min(cfg.local_buffer, prompt_len - s0)
    W = cfg.block_size
    nsealed = (buf0 - s0) // W
    blocks = []
    for b in range(nsealed + 1):
        lo = s0 + b * W
        hi = lo + W if b < nsealed else buf0
        blocks.append(BlockO(lo, hi, _cluster_span(keys, values, lo, hi, cfg, block_seed(cfg.seed, head, b))))
    led = LedgerO(s0, blocks, buf0, prompt_len)
    if cfg.hierarchy is not None:
        for b, blk in enumerate(led.blocks):
            blk.coarse = coarse_level(blk.fine, cfg, blk.end - blk.start, block_seed(cfg.seed, head, b, 1))
    return led


def _settle(blk: BlockO, keys, values) -> None:
    """Lloyd(min_iters=0) from the current centroids over the block's members (clustering.py:343-356)."""
    if blk.fine.k == 0:
        return
    ids = np.sort(np.concatenate(blk.fine.members))
    c, lab = lloyd(np.asarray(keys, dtype=np.float64)[ids], blk.fine.kc, 0)
    blk.fine = compact(c, lab, ids)
    value_means(blk.fine, values)


def split_final(led: LedgerO, keys, values, cfg: EngineConfig, head: int, settle: bool = True) -> None:
    """While |final| >= W + alpha seal its first W tokens; straddlers split with np.mean
    centroids, then both sides are settled (clustering.py:359-401)."""
    W = cfg.block_size
    k64 = np.asarray(keys, dtype=np.float64)
    v64 = np.asarray(values, dtype=np.float64)
    while led.final.end - led.final.start >= W + cfg.alpha:
        old = led.final
        cut = old.start + W
        sides = ([], [], []), ([], [], [])  # (kc, vc, members) for left / right
        for j, mem in enumerate(old.fine.members):
            parts = (mem[mem < cut], mem[mem >= cut])
            for part, (kcs, vcs, ms) in zip(parts, sides):
                if not part.size:
                    continue
                if part.size == mem.size:
                    kcs.append(old.fine.kc[j]); vcs.append(old.fine.vc[j]); ms.append(mem)
                else:
                    kcs.append(np.mean(k64[part], axis=0)); vcs.append(np.mean(v64[part], axis=0))
                    ms.append(part.copy())
        d = k64.shape[1]

        def mk(t):
            return Level(np.stack(t[0]) if t[0] else np.zeros((0, d)),
                         np.stack(t[1]) if t[1] else np.zeros((0, d)), t[2])

        sealed = BlockO(old.start, cut, mk(sides[0]))
        led.blocks[-1] = sealed
        led.blocks.append(BlockO(cut, old.end, mk(sides[1])))
        led.splits += 1
        if settle:
            _settle(sealed, keys, values)
            _settle(led.final, keys, values)
        if cfg.hierarchy is not None:
            sealed.coarse = coarse_level(sealed.fine, cfg, W,
                                         block_seed(cfg.seed, head, len(led.blocks) - 2, 2))


def append_update(led: LedgerO, keys, values, cfg: EngineConfig, rng, head: int = 0) -> LedgerO:
    """Absorb the oldest L buffered tokens into the final block (clustering.py:404-472)."""
    L = cfg.local_buffer
    if led.buffer_len < 2 * L:
        raise RuntimeError(f"buffer underflow: have {led.buffer_len} tokens, need {2 * L}")
    k64 = np.asarray(keys, dtype=np.float64)
    new = np.arange(led.buffer_start, led.buffer_start + L, dtype=np.int64)
    fin = led.final
    # (1) seeds: existing final centroids, then ceil(L/r) sampled appended tokens
    samp = rng.choice(L, size=-(-L // cfg.fine_ratio), replace=False)
    cen = np.concatenate([fin.fine.kc, k64[new[samp]]], axis=0)
    cnt = np.concatenate([fin.fine.sizes, np.zeros(samp.size, dtype=np.int64)])
    # (2) single pass, running-mean sequential assignment (direct-form distances)
    for t in new:
        x = k64[t]
        j = int(np.argmin(np.einsum("kd,kd->k", cen - x, cen - x)))
        cnt[j] += 1
        cen[j] += (x - cen[j]) / cnt[j]
    # (3) Lloyd refinement over the whole final block + appended tokens
    ids = np.sort(np.concatenate(fin.fine.members + [new]) if fin.fine.members else new)
    c, lab = lloyd(k64[ids], cen, cfg.refine_kmeans_iters)
    lev = compact(c, lab, ids)
    value_means(lev, values)                                           # (4)
    led.blocks[-1] = BlockO(fin.start, int(new[-1]) + 1, lev)
    led.buffer_start += L
    split_final(led, keys, values, cfg, head)                          # (5)
    if cfg.hierarchy is not None:                                      # (6)
        f = led.final
        f.coarse = coarse_level(f.fine, cfg, f.end - f.start,
                                block_seed(cfg.seed, head, led.buffer_start, 3))
    return led


# Positional comparator (clustering.py:479-541) -- contiguous r-token pages.


def _pages(keys, values, lo, hi, r) -> Level:
    k64 = np.asarray(keys, dtype=np.float64)
    v64 = np.asarray(values, dtype=np.float64)
    mem = [np.arange(s, min(s + r, hi), dtype=np.int64) for s in range(lo, hi, r)]
    d = k64.shape[1]
    if not mem:
        return empty_level(d)
    return Level(np.stack([np.mean(k64[m], axis=0) for m in mem]),
                 np.stack([np.mean(v64[m], axis=0) for m in mem]), mem)


def positional_ledger(keys, values, prompt_len: int, cfg: EngineConfig) -> LedgerO:
    if prompt_len <= cfg.sink_tokens:
        raise ConfigError(f"prompt_len {prompt_len} must exceed sink_tokens {cfg.sink_tokens}")
    s0 = cfg.sink_tokens
    buf0 = prompt_len - min(cfg.local_buffer, prompt_len - s0)
    W = cfg.block_size
    nsealed = (buf0 - s0) // W
    blocks = []
    for b in range(nsealed + 1):
        lo = s0 + b * W
        hi = lo + W if b < nsealed else buf0
        blocks.append(BlockO(lo, hi, _pages(keys, values, lo, hi, cfg.fine_ratio)))
    return LedgerO(s0, blocks, buf0, prompt_len)


def positional_update(led: LedgerO, keys, values, cfg: EngineConfig) -> LedgerO:
    L = cfg.local_buffer
    if led.buffer_len < 2 * L:
        raise RuntimeError("buffer underflow")
    hi = led.buffer_start + L
    led.blocks[-1] = BlockO(led.final.start, hi, _pages(keys, values, led.final.start, hi, cfg.fine_ratio))
    led.buffer_start += L
    split_final(led, keys, values, cfg, 0, settle=False)
    return led


# ---------------------------------------------------------------------------
# Streaming-softmax partials (attention.py:22-68, 230-239)


@dataclass
class Partial:
    m: float
    s: float
    a: np.ndarray

    @staticmethod
    def empty(d: int) -> "Partial":
        return Partial(-np.inf, 0.0, np.zeros(d))

    def out(self) -> np.ndarray:
        if self.s <= 0.0:
            raise ValueError("cannot finalize an empty partial")
        return self.a / self.s


def partial_of(logits, vals, weights=None) -> Partial:
    lg = np.asarray(logits, dtype=np.float64)
    if lg.size == 0:
        return Partial.empty(np.asarray(vals).shape[-1])
    m = float(np.max(lg))
    w = np.exp(lg - m)
    if weights is not None:
        w = w * np.asarray(weights, dtype=np.float64)
    return Partial(m, float(np.sum(w)), w @ np.asarray(vals, dtype=np.float64))


def merge(parts) -> Partial:
    live = [p for p in parts if p.s != 0.0]
    if not live:
        raise ValueError("all partials are empty")
    m = max(p.m for p in live)
    return Partial(m, float(sum(p.s * np.exp(p.m - m) for p in live)),
                   sum(p.a * np.exp(p.m - m) for p in live))


def exact_part(q, qpos: int, keys, vals, pos, d: int, theta: float) -> Partial:
    """True-position rotation of q and keys, 1/sqrt(d) logits (attention.py:71-87)."""
    k64 = np.asarray(keys, dtype=np.float64)
    if k64.shape[0] == 0:
        return Partial.empty(d)
    lg = rotate(k64, np.asarray(pos), d, theta) @ rotate(q, qpos, d, theta) / np.sqrt(d)
    return partial_of(lg, vals)


def dense_attention(q, qpos, keys, vals, pos, d, theta) -> np.ndarray:
    if np.asarray(keys).shape[0] == 0:
        raise ValueError("exact attention over an empty key set")
    return exact_part(q, qpos, keys, vals, pos, d, theta).out()


# ---------------------------------------------------------------------------
# Lookup + selection (attention.py:144-375)


def group_scores(qlk: np.ndarray, kc: np.ndarray, sizes: np.ndarray, d: int):
    """Eq. 1 per head normalised by sum N*e, averaged over the GQA group (attention.py:267-290).
    Returns (mean scores (K,), logits (G, K))."""
    lg = np.asarray(qlk, dtype=np.float64) @ kc.T / np.sqrt(d)
    e = np.exp(lg - np.max(lg, axis=1, keepdims=True))
    sc = e / (e @ sizes.astype(np.float64))[:, None]
    return np.mean(sc, axis=0), lg


def budget_select(scores, sizes, budget: int, tie_keys=None):
    """Greedy take-while-cum<budget in (score desc, tie_key asc) order; the crossing cluster is
    included (attention.py:192-207).  Returns (selected positions, rejected positions), each
    in visiting order."""
    if budget < 0:
        raise ValueError("budget must be >= 0")
    n = len(scores)
    keys = range(n) if tie_keys is None else tie_keys
    order = sorted(range(n), key=lambda i: (-float(scores[i]), keys[i]))
    sel, rej, cum = [], [], 0
    for i in order:
        if cum < budget:
            sel.append(i)
            cum += int(sizes[i])
        else:
            rej.append(i)
    return sel, rej


@dataclass
class Lookup:
    sel_idx: np.ndarray            # sorted selected token ids
    sel_refs: list                 # (block, cluster, 2)
    fine_rej: list                 # (ref, vc row, size, logits (G,))
    coarse_rej: list
    scored: int
    rejected: int


def _flat(led: LedgerO, coarse: bool):
    """Concatenate one level over blocks in ref order; returns kc, vc, sizes, members, refs."""
    kcs, vcs, mem, refs = [], [], [], []
    for b, blk in enumerate(led.blocks):
        lev = blk.coarse if coarse else blk.fine
        if lev is None:
            continue
        for j in range(lev.k):
            refs.append((b, j, 1 if coarse else 2))
        kcs.append(lev.kc); vcs.append(lev.vc); mem.extend(lev.members)
    d = led.blocks[0].fine.kc.shape[1]
    if not refs:
        return np.zeros((0, d)), np.zeros((0, d)), np.zeros(0, np.int64), [], []
    return (np.concatenate(kcs), np.concatenate(vcs),
            np.array([m.size for m in mem], np.int64), mem, refs)


def flat_lookup(qlk, led: LedgerO, cfg: EngineConfig, d: int) -> Lookup:
    qlk = np.atleast_2d(qlk)
    kc, vc, sz, mem, refs = _flat(led, False)
    if not refs:
        raise ConfigError("ledger has no clusters")
    sc, lg = group_scores(qlk, kc, sz, d)
    sel, rej = budget_select(sc, sz, cfg.token_budget, refs)
    sel_idx = np.sort(np.concatenate([mem[i] for i in sel])) if sel else np.zeros(0, np.int64)
    fr = [(refs[i], vc[i], int(sz[i]), lg[:, i]) for i in rej]
    return Lookup(sel_idx, [refs[i] for i in sel], fr, [], len(refs), len(fr))


def hier_lookup(qlk, led: LedgerO, cfg: EngineConfig, d: int) -> Lookup:
    """Promote coarse clusters to ceil(p * total) tokens, then select fine children with a
    denominator over {promoted fine} U {rejected coarse} (attention.py:293-351)."""
    if cfg.hierarchy is None:
        raise ConfigError("hierarchical lookup requires hierarchy enabled")
    qlk = np.atleast_2d(qlk)
    ckc, cvc, csz, _, crefs = _flat(led, True)
    if not crefs:
        raise ConfigError("ledger has no coarse clusters")
    sc1, lg1 = group_scores(qlk, ckc, csz, d)
    promo, crej = budget_select(sc1, csz, int(np.ceil(cfg.hierarchy.promote_fraction * int(csz.sum()))), crefs)
    fkc, fvc, fsz, fmem, frefs = [], [], [], [], []
    for i in promo:
        b, j, _ = crefs[i]
        fine = led.blocks[b].fine
        for ch in led.blocks[b].coarse.children[j]:
            fkc.append(fine.kc[ch]); fvc.append(fine.vc[ch]); fsz.append(fine.members[ch].size)
            fmem.append(fine.members[ch]); frefs.append((b, ch, 2))
    nf = len(frefs)
    ukc = np.stack(fkc + [ckc[i] for i in crej])
    usz = np.array(fsz + [int(csz[i]) for i in crej], np.int64)
    sc2, lg2 = group_scores(qlk, ukc, usz, d)
    sel, rej = budget_select(sc2[:nf], usz[:nf], cfg.token_budget, frefs)
    sel_idx = np.sort(np.concatenate([fmem[i] for i in sel])) if sel else np.zeros(0, np.int64)
    fr = [(frefs[i], fvc[i], int(fsz[i]), lg2[:, i]) for i in rej]
    cr = [(crefs[i], cvc[i], int(csz[i]), lg1[:, i]) for i in crej]
    return Lookup(sel_idx, [frefs[i] for i in sel], fr, cr, len(crefs) + nf, len(fr) + len(cr))


def replacement(gi: int, rej: list, d: int) -> Partial:
    """Eq. 2: weights N*exp(logit) on value centroids, logits reused (attention.py:210-227)."""
    if not rej:
        return Partial.empty(d)
    lg = np.array([r[3][gi] for r in rej])
    return partial_of(lg, np.stack([r[1] for r in rej]), weights=np.array([r[2] for r in rej], np.float64))


# ---------------------------------------------------------------------------
# Decode step + pipeline (attention.py:410-552, pipeline.py:69-220)


@dataclass
class HeadStat:
    selected_refs: list
    selected_tokens: int
    scored_centroids: int
    rejected_centroids: int


@dataclass
class StepReport:
    step: int
    per_head: list
    cache_len: int
    sink_count: int
    buffer_len: int
    num_kv_heads: int
    selected_indices: list = field(default_factory=list)
    update_occurred: bool = False
    mode: str = "multipole"
    outputs: np.ndarray | None = None


def decode_step(queries, ledgers, keys, values, cache_len, step, cfg: EngineConfig,
                layout: HeadLayout, mode="multipole", rot_keys=None):
    """`rot_keys` (test hook, per head (T, d)): use these already-rotated keys for the exact
    logits instead of rotating `keys` -- emulates a cache that stores K_rot in a lower precision."""
    d = layout.head_dim
    th = cfg.rope_theta
    out = np.empty((layout.num_q_heads, d))
    stats, sels = [], []
    use_rep = mode != "flat-no-replacement"
    for h, led in enumerate(ledgers):
        grp = list(layout.q_heads_of(h))
        qlk = np.stack([lookup_query(queries[g], cfg, d) for g in grp])
        lk = hier_lookup(qlk, led, cfg, d) if cfg.hierarchy is not None else flat_lookup(qlk, led, cfg, d)
        sinks = np.arange(0, min(led.sink_end, cache_len), dtype=np.int64)
        buf = np.arange(led.buffer_start, cache_len, dtype=np.int64)
        K, V = keys[h], values[h]
        for gi, g in enumerate(grp):
            q = queries[g]
            if rot_keys is None:
                parts = [exact_part(q, cache_len, K[ix], V[ix], ix, d, th) for ix in (sinks, buf, lk.sel_idx)]
            else:
                qr = rotate(q, cache_len, d, th)
                parts = [partial_of(np.asarray(rot_keys[h][ix], np.float64) @ qr / np.sqrt(d), V[ix]) if ix.size
                         else Partial.empty(d) for ix in (sinks, buf, lk.sel_idx)]
            if use_rep:
                parts += [replacement(gi, r, d) for r in (lk.fine_rej, lk.coarse_rej) if r]
            out[g] = merge(parts).out()
        sels.append(lk.sel_idx)
        stats.append(HeadStat(lk.sel_refs, int(lk.sel_idx.size), lk.scored, lk.rejected if use_rep else 0))
    rep = StepReport(step, stats, cache_len, min(cfg.sink_tokens, cache_len),
                     cache_len - ledgers[0].buffer_start, layout.num_kv_heads, sels, mode=mode)
    return out, rep


class Store:
    """Growable fp32 (T, d) store with doubling capacity (pipeline.py:26-52)."""

    def __init__(self, arr):
        arr = np.asarray(arr, np.float32)
        self.buf = np.zeros((max(16, 2 * arr.shape[0]), arr.shape[1]), np.float32)
        self.buf[: arr.shape[0]] = arr
        self.n = arr.shape[0]

    def push(self, row):
        if self.n == self.buf.shape[0]:
            self.buf = np.concatenate([self.buf, np.zeros_like(self.buf)])
        self.buf[self.n] = row
        self.n += 1

    @property
    def data(self):
        return self.buf[: self.n]


@dataclass
class StateO:
    trace: KvTrace
    cfg: EngineConfig
    mode: str
    ledgers: list
    kstore: list         # per kv-head Store
    vstore: list
    cursor: int = 0

    @property
    def cache_len(self) -> int:
        return self.trace.prompt_len + self.cursor

    @property
    def keys(self):
        return [s.data for s in self.kstore]

    @property
    def values(self):
        return [s.data for s in self.vstore]


def prefill(trace: KvTrace, cfg: EngineConfig, mode="multipole", ledgers=None) -> StateO:
    """`ledgers` may be supplied (e.g. converted from a device ledger) to skip clustering."""
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    P = trace.prompt_len
    ks = [trace.keys[h, :P].copy() for h in range(trace.layout.num_kv_heads)]
    vs = [trace.values[h, :P].copy() for h in range(trace.layout.num_kv_heads)]
    if ledgers is None:
        if mode == "oracle":
            ledgers = []
        elif mode == "positional-baseline":
            ledgers = [positional_ledger(k, v, P, cfg) for k, v in zip(ks, vs)]
        else:
            ledgers = [prefill_ledger(k, v, P, cfg, h) for h, (k, v) in enumerate(zip(ks, vs))]
    return StateO(trace, cfg, mode, ledgers, [Store(k) for k in ks], [Store(v) for v in vs])


def step(st: StateO, queries, new_keys, new_values):
    cfg, lay = st.cfg, st.trace.layout
    d, n = lay.head_dim, st.cache_len
    if st.mode == "oracle":
        pos = np.arange(n, dtype=np.int64)
        out = np.empty((lay.num_q_heads, d))
        for h in range(lay.num_kv_heads):
            for g in lay.q_heads_of(h):
                out[g] = dense_attention(queries[g], n, st.keys[h][:n], st.values[h][:n], pos, d, cfg.rope_theta)
        rep = StepReport(st.cursor, [], n, 0, 0, lay.num_kv_heads, mode="oracle")
    else:
        out, rep = decode_step(queries, st.ledgers, st.keys, st.values, n, st.cursor, cfg, lay, st.mode)
    for h in range(lay.num_kv_heads):
        st.kstore[h].push(new_keys[h])
        st.vstore[h].push(new_values[h])
        if st.ledgers:
            st.ledgers[h].total += 1
    if st.ledgers and st.ledgers[0].buffer_len >= 2 * cfg.local_buffer:
        for h in range(lay.num_kv_heads):
            if st.mode == "positional-baseline":
                positional_update(st.ledgers[h], st.keys[h], st.values[h], cfg)
            else:
                append_update(st.ledgers[h], st.keys[h], st.values[h], cfg, update_rng(cfg.seed, st.cursor, h), h)
        rep.update_occurred = True
    st.cursor += 1
    return out, rep


def run(trace: KvTrace, cfg: EngineConfig, mode="multipole", max_steps=None):
    if trace.decode_steps < 1:
        raise ValueError("trace has no decode steps")
    st = prefill(trace, cfg, mode)
    n = trace.decode_steps if max_steps is None else min(max_steps, trace.decode_steps)
    reps = []
    for t in range(n):
        p = trace.prompt_len + t
        out, rep = step(st, trace.queries[:, t], trace.keys[:, p], trace.values[:, p])
        rep.outputs = out
        reps.append(rep)
    return reps


# ---------------------------------------------------------------------------
# Checkers: ledger audit (clustering.py:548-623) and memory-op counts (bench.py:53-71)


class AuditError(AssertionError):
    pass


def audit(led: LedgerO, keys, cfg: EngineConfig, values=None, rel_tol=1e-5, check_assignment=True) -> None:
    k64 = np.asarray(keys, dtype=np.float64)
    toks = [np.arange(led.sink_end, dtype=np.int64)]
    for blk in led.blocks:
        toks.extend(blk.fine.members)
    toks.append(np.arange(led.buffer_start, led.total, dtype=np.int64))
    allt = np.sort(np.concatenate(toks))
    if allt.size != led.total or not np.array_equal(allt, np.arange(led.total)):
        raise AuditError("token indices do not tile [0, total) exactly")
    at = led.sink_end
    for blk in led.blocks[:-1]:
        if blk.start != at or blk.end - blk.start != cfg.block_size:
            raise AuditError("sealed block spans are not contiguous W-sized")
        at = blk.end
    if led.final.start != at or led.final.end != led.buffer_start:
        raise AuditError("final block span inconsistent with buffer start")
    flen = led.final.end - led.final.start
    if flen > cfg.block_size + cfg.alpha:
        raise AuditError("final block exceeds W + alpha")
    if led.splits > 0 and flen < cfg.alpha:
        raise AuditError("final block shorter than alpha after a split")
    v64 = None if values is None else np.asarray(values, dtype=np.float64)
    for blk in led.blocks:
        lev = blk.fine
        if lev.k == 0:
            continue
        idx = np.concatenate(lev.members)
        own = np.concatenate([np.full(m.size, j) for j, m in enumerate(lev.members)])
        if idx.min() < blk.start or idx.max() >= blk.end:
            raise AuditError("cluster member outside its block span")
        cnt = lev.sizes.astype(np.float64)[:, None]
        for cen, src in ((lev.kc, k64), (lev.vc, v64)):
            if src is None:
                continue
            acc = np.zeros_like(cen)
            np.add.at(acc, own, src[idx])
            if np.max(np.abs(acc / cnt - cen)) > rel_tol * max(1.0, float(np.max(np.abs(cen)))):
                raise AuditError("centroid drifted from member mean")
        if check_assignment and not np.array_equal(assign_nearest(k64[idx], lev.kc), own):
            raise AuditError("a member is not assigned to its nearest centroid")


def memops(rep: StepReport) -> dict:
    """Vector-load counts of one step (bench.py:53-71)."""
    base = 2 * rep.cache_len * rep.num_kv_heads
    if rep.mode == "oracle" or not rep.per_head:
        return dict(total=0, baseline=base, ratio=0.0)
    kc = sum(h.scored_centroids for h in rep.per_head)
    vc = sum(h.rejected_centroids for h in rep.per_head)
    sel = sum(h.selected_tokens for h in rep.per_head)
    tot = kc + vc + 2 * sel + 2 * rep.sink_count * rep.num_kv_heads + 2 * rep.buffer_len * rep.num_kv_heads
    return dict(key_centroid=kc, value_centroid=vc, exact=2 * sel, total=tot, baseline=base, ratio=tot / base)


def ledger_arrays(led: LedgerO) -> dict:
    """Flatten a ledger to plain arrays (spans, sizes, members, centroids, children) so two
    ledgers -- oracle, reference or device -- can be compared with array_equal."""
    out = {"meta": np.array([led.sink_end, led.buffer_start, led.total, led.splits, len(led.blocks)], np.int64),
           "spans": np.array([[b.start, b.end] for b in led.blocks], np.int64).reshape(-1, 2)}
    for lv in ("fine", "coarse"):
        levs = [getattr(b, lv) for b in led.blocks]
        if any(x is None for x in levs):
            continue
        out[lv + "_counts"] = np.array([x.k for x in levs], np.int64)
        out[lv + "_sizes"] = np.concatenate([x.sizes for x in levs])
        mem = [m for x in levs for m in x.members]
        out[lv + "_members"] = np.concatenate(mem) if mem else np.zeros(0, np.int64)
        out[lv + "_kc"] = np.concatenate([x.kc.reshape(-1, x.kc.shape[-1]) for x in levs])
        out[lv + "_vc"] = np.concatenate([x.vc.reshape(-1, x.kc.shape[-1]) for x in levs])
        if lv == "coarse":
            kids = [np.asarray(c, np.int64) for x in levs for c in x.children]
            out["coarse_children"] = np.concatenate(kids) if kids else np.zeros(0, np.int64)
    return out
