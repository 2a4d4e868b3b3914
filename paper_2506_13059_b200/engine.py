"""Device-resident Multipole Attention decode engine (one attention layer, a batch of sequences).

This is the B200 replacement for the per-kv-head Python loops of the reference
(attention.py:410-552 `decode_step_attention`, pipeline.py:124-191 `step`).  All state lives
in HBM; one decode step is a short, graph-capturable chain of libmpattn kernels on one stream:

    mpa_rotate_queries   q -> q_rot (true position, fp32) and q_lookup (Delta, fp64)     K1
    mpa_centroid_logits  fp64 logits of the fine (or coarse) centroids                   K9
    mpa_select           Eq. 1 scores + size-weighted radix select to the budget         K10
    [hierarchy: mpa_hier_candidates, mpa_centroid_logits (fine children), mpa_select with
     the coarse-rejected union denominator]
    (work lists)         sinks ++ buffer ++ selected members; rejected centroids + ln N
    mpa_sparse_decode    gather + exact attention + centroid replacement, split-KV merge K11+K12

Attention happens before the step's token is appended (pipeline.py:137-159); the online
cluster update runs when the buffer reaches 2L (pipeline.py:161) -- see clustering.py.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from ._lib import MpaCache, call, dtype_code, ptr, stream_ptr
from .core import ConfigError, EngineConfig, HeadLayout, inv_freq
from .ledger import DeviceLedgers, HostLedger



class DecodeEngine:
    def __init__(self, cfg: EngineConfig, layout: HeadLayout, n_seq: int, tcap: int,
                 dtype: torch.dtype = torch.bfloat16, device="cuda", kcap: int | None = None,
                 ccap: int | None = None, mode: str = "multipole", use_graphs: bool | None = None,
                 page_size: int | None = None, n_pages: int | None = None, page_order: str = "sequential"):
        """page_size: serve K_rot / V from a paged pool (pipeline.py:26-52 `_KvStore` as the
        block-table cache of a paged server): pools [n_pages, Hkv, page_size, d] (HND block layout:
        a head's tokens contiguous inside a page), one block table row per sequence, pages taken
        from a free list as sequences grow
        ("shuffled" hands them out in random order, as a long-running server would).  K_raw, the
        clustering view, stays [L, tcap, d]."""
        if not torch.cuda.is_available():
            raise RuntimeError("DecodeEngine needs a CUDA device (B200); there is no CPU fallback")
        _lib.lib()  # fail loudly if libmpattn.so is missing
        self.cfg, self.layout, self.mode = cfg, layout, mode
        self.n_seq, self.d, self.G = n_seq, layout.head_dim, layout.group_size
        self.Hkv, self.Hq = layout.num_kv_heads, layout.num_q_heads
        self.L = n_seq * self.Hkv
        self.tcap, self.dtype = tcap, dtype
        self.device = torch.device(device)
        self._dev_idx = self.device.index if self.device.index is not None else torch.cuda.current_device()
        r = cfg.fine_ratio
        self.kcap = kcap or max(64, 2 * (tcap // r) + 64)
        hier = cfg.hierarchy is not None
        self.ccap = ccap or (max(16, 2 * (tcap // cfg.hierarchy.r1) + 64) if hier else 0)
        L, d, G, dev = self.L, self.d, self.G, self.device
        z = dict(device=dev)
        self.k_raw = torch.zeros(L, tcap, d, dtype=dtype, **z)
        self.page_size = page_size
        if page_size is None:
            self.k_rot = torch.zeros(L, tcap, d, dtype=dtype, **z)
            self.v = torch.zeros(L, tcap, d, dtype=dtype, **z)
            self.block_table = None
        else:
            if page_size < 1 or page_size & (page_size - 1):
                raise ConfigError(f"page_size {page_size} must be a power of two")
            self.pages_per_seq = -(-tcap // page_size)
            self.n_pages = n_pages or n_seq * self.pages_per_seq
            self.k_rot = torch.zeros(self.n_pages, self.Hkv, page_size, d, dtype=dtype, **z)
            self.v = torch.zeros(self.n_pages, self.Hkv, page_size, d, dtype=dtype, **z)
            self.block_table = torch.zeros(n_seq, self.pages_per_seq, dtype=torch.int32, **z)
            self._bt_host = np.full((n_seq, self.pages_per_seq), -1, np.int64)
            free = np.arange(self.n_pages)
            if page_order == "shuffled":
                free = np.random.default_rng(cfg.seed).permutation(free)
            self._free_pages = list(free[::-1])  # pop() hands out free[0] first
        self.led = DeviceLedgers(L, d, tcap, self.kcap, self.ccap, dtype, hier, dev)
        self.inv_freq = torch.as_tensor(inv_freq(d, cfg.rope_theta), dtype=torch.float64, device=dev)
        # (cos, sin) of the lookup view's fixed angles delta * inv_freq (rope.py:66-68, numpy like the
        # reference): lets the logits kernel rotate the queries itself
        ang = float(cfg.window_offset) * inv_freq(d, cfg.rope_theta)
        self.cs_lk = torch.as_tensor(np.stack([np.cos(ang), np.sin(ang)], axis=-1), dtype=torch.float64, device=dev)
        # per-sequence scalars (host mirror + device copy)
        self.cache_len = np.zeros(n_seq, np.int64)
        self.sink_end = np.zeros(n_seq, np.int64)
        self.buffer_start = np.zeros(n_seq, np.int64)
        self.splits = np.zeros(L, np.int64)
        self.cache_len_d = torch.zeros(n_seq, dtype=torch.int32, **z)
        self.sink_end_d = torch.zeros(n_seq, dtype=torch.int32, **z)
        self.buffer_start_d = torch.zeros(n_seq, dtype=torch.int32, **z)
        self.ntok_dense_d = torch.zeros(L, dtype=torch.int32, **z)
        self.append_ticket = torch.zeros(1, dtype=torch.int32, **z)
        # workspace
        self.q_rot = torch.zeros(n_seq, self.Hq, d, dtype=torch.float32, **z)
        self.q_lk = torch.zeros(n_seq, self.Hq, d, dtype=torch.float64, **z)
        self.logits = torch.zeros(L, G, self.kcap, dtype=torch.float64, **z)
        self.elocal = torch.zeros(L, G, self.kcap, dtype=torch.float64, **z)
        self.flag = torch.zeros(L, self.kcap, dtype=torch.uint8, **z)
        self.sel_tokens = torch.zeros(L, dtype=torch.int32, **z)
        self.cstats = torch.zeros(L, -(-self.kcap // 128), G, 2, dtype=torch.float64, **z)
        self.budget = torch.full((L,), cfg.token_budget, dtype=torch.int64, **z)
        if hier:
            self.clogits = torch.zeros(L, G, self.ccap, dtype=torch.float64, **z)
            self.celocal = torch.zeros(L, G, self.ccap, dtype=torch.float64, **z)
            self.cflag = torch.zeros(L, self.ccap, dtype=torch.uint8, **z)
            self.cbudget = torch.zeros(L, dtype=torch.int64, **z)
            self.cand = torch.zeros(L, self.kcap, dtype=torch.int32, **z)
            self.n_cand = torch.zeros(L, dtype=torch.int32, **z)
            self.csel_tokens = torch.zeros(L, dtype=torch.int32, **z)
            self.ccstats = torch.zeros(L, -(-self.ccap // 128), G, 2, dtype=torch.float64, **z)
        self.tok_cap = tcap
        self.rej_cap = self.kcap + self.ccap
        self.tok = torch.zeros(L, self.tok_cap, dtype=torch.int32, **z)
        self.rej = torch.zeros(L, self.rej_cap, dtype=torch.int32, **z)
        self.rej_w = torch.zeros(L, self.rej_cap, 4 if G <= 4 else 8, dtype=torch.float32, **z)
        self.stats = torch.zeros(4, L, dtype=torch.int32, **z)
        self.ws = torch.zeros(0, dtype=torch.uint8, **z)  # fused-kernel workspace (grown on demand)
        self.out = torch.zeros(n_seq, self.Hq, d, dtype=torch.float32, **z)
        if self.block_table is None:
            self.cache_struct = MpaCache(ptr(self.k_rot), ptr(self.k_raw), ptr(self.v), dtype_code(dtype), L, tcap, d,
                                         None, 0, 0, 0, self.Hkv)
        else:
            self.cache_struct = MpaCache(ptr(self.k_rot), ptr(self.k_raw), ptr(self.v), dtype_code(dtype), L, tcap, d,
                                         ptr(self.block_table), page_size, self.pages_per_seq, self.n_pages, self.Hkv)
        self.last_split = 1
        self.cursor = 0
        # the flat serving path (fused_lookup_path) hands the fused kernel a contiguous-centroid
        # list: every centroid's replacement weight in id order, the selected ones -inf
        self.use_graphs = True if use_graphs is None else use_graphs
        self._graph = None
        self._gexec = None  # its cudaGraphExec_t (mpa_step_host)
        self._graph_raw = None  # its cudaGraph_t, kept for mpa_decode_step_rebind (flat path)
        self._bound = None
        self.n_captures = 0  # step-graph captures so far (bench reports it)
        self.time_fused = False  # bench: CUDA events around the fused kernel inside the step graph
        self._fev = None
        self.last_lloyd_rounds = 0
        self.last_update: dict | None = None

    # ------------------------------------------------------------------ KV cache
    def reserve(self, n: int) -> None:
        """Capacity for n more tokens in every sequence: the logical bound, and (paged) the pages
        they land in, taken from the free list and published in the block table."""
        if int(self.cache_len.max()) + n > self.tcap:
            raise RuntimeError(f"KV cache capacity {self.tcap} exceeded")
        if self.block_table is None:
            return
        ps, new = self.page_size, []
        for s in range(self.n_seq):
            for pg in range(int(self.cache_len[s]) // ps, -(-(int(self.cache_len[s]) + n) // ps)):
                if self._bt_host[s, pg] < 0:
                    if not self._free_pages:
                        raise RuntimeError(f"KV page pool of {self.n_pages} pages exhausted")
                    self._bt_host[s, pg] = self._free_pages.pop()
                    new.append((s, pg))
        if new:
            s_i, p_i = zip(*new)
            self.block_table[list(s_i), list(p_i)] = torch.as_tensor(self._bt_host[list(s_i), list(p_i)],
                                                                      dtype=torch.int32, device=self.device)

    def kv_rows(self, l: int, t) -> torch.Tensor:
        """Rows of tokens t (int64 tensor or array) of ledger l in k_rot / v viewed as [-1, d]."""
        t = torch.as_tensor(t, dtype=torch.int64, device=self.device)
        if self.block_table is None:
            return l * self.tcap + t
        s, h, ps = l // self.Hkv, l % self.Hkv, self.page_size
        page = self.block_table[s].to(torch.int64)[t // ps]
        return (page * self.Hkv + h) * ps + t % ps

    def values(self, l: int, t) -> torch.Tensor:
        """Cached values of tokens t of ledger l, [len(t), d] in the cache dtype."""
        return self.v.view(-1, self.d)[self.kv_rows(l, t)]

    def keys_rotated(self, l: int, t) -> torch.Tensor:
        return self.k_rot.view(-1, self.d)[self.kv_rows(l, t)]

    def write_tokens(self, k: torch.Tensor, v: torch.Tensor, pos0: torch.Tensor | None = None) -> None:
        """Write n new tokens per ledger: k, v fp32 [n_seq, Hkv, n, d] (device) at cache_len."""
        n = k.shape[2]
        k = k.reshape(self.L, n, self.d).float().contiguous()
        v = v.reshape(self.L, n, self.d).float().contiguous()
        if pos0 is None:
            self.reserve(n)
            # positions and the length counters advance on the device (one launch)
            call("mpa_kv_append", self.cache_struct, ptr(k), ptr(v), self.Hkv, n, ptr(self.cache_len_d),
                 ptr(self.ntok_dense_d), ptr(self.inv_freq), ptr(self.append_ticket), stream_ptr())
        else:
            if self.block_table is not None:
                raise ConfigError("explicit write positions need a flat cache")
            call("mpa_kv_write", self.cache_struct, ptr(k), ptr(v), ptr(pos0), n, ptr(self.inv_freq), stream_ptr())
            self.cache_len_d += n
            self.ntok_dense_d += n
        self.cache_len += n

    def set_prompt_layout(self) -> None:
        """Sinks / buffer split of the prompt (clustering.py:295-299)."""
        cfg = self.cfg
        for s in range(self.n_seq):
            P = int(self.cache_len[s])
            if P <= cfg.sink_tokens:
                raise ConfigError(f"prompt_len {P} must exceed sink_tokens {cfg.sink_tokens}")
            self.sink_end[s] = cfg.sink_tokens
            self.buffer_start[s] = P - min(cfg.local_buffer, P - cfg.sink_tokens)
        self._sync_scalars()

    def _sync_scalars(self) -> None:
        self.sink_end_d.copy_(torch.as_tensor(self.sink_end, dtype=torch.int32))
        self.buffer_start_d.copy_(torch.as_tensor(self.buffer_start, dtype=torch.int32))
        self.cache_len_d.copy_(torch.as_tensor(self.cache_len, dtype=torch.int32))
        self.ntok_dense_d.copy_(torch.as_tensor(np.repeat(self.cache_len, self.Hkv), dtype=torch.int32))
        if self.cfg.hierarchy is not None:
            p = self.cfg.hierarchy.promote_fraction
            clustered = np.repeat(self.buffer_start - self.sink_end, self.Hkv)
            self.cbudget.copy_(torch.as_tensor([int(np.ceil(p * int(c))) for c in clustered], dtype=torch.int64))

    def load_ledgers(self, ledgers: list[HostLedger]) -> None:
        for l, h in enumerate(ledgers):
            self.led.load(l, h)
            s = l // self.Hkv
            self.sink_end[s], self.buffer_start[s] = h.sink_end, h.buffer_start
            self.splits[l] = h.splits
        self._sync_scalars()

    # ------------------------------------------------------------------ decode
    def _workspace(self, n_split: int) -> torch.Tensor:
        """Zero-filled workspace of mpa_sparse_decode (partials + per-ledger tickets)."""
        need = int(_lib.lib().mpa_sparse_decode_workspace(self.L, self.G, self.d, dtype_code(self.dtype), n_split))
        if self.ws.numel() < need:
            self.ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
        return self.ws

    def rotate(self, q: torch.Tensor, exact: bool = True, lookup: bool = True) -> None:
        """Exact view q_rot (at cache_len) and / or lookup view q_lk (at the window offset)."""
        q = q.float().contiguous()
        call("mpa_rotate_queries", ptr(q), self.n_seq, self.Hq, self.d, ptr(self.cache_len_d), self.cfg.window_offset,
             ptr(self.inv_freq), 1.0 / math.sqrt(self.d), ptr(self.q_rot) if exact else None,
             ptr(self.q_lk) if lookup else None, stream_ptr())

    def _cluster_bounds(self):
        """Per-ledger cluster-count bounds passed to the lookup kernels (grid / smem sizing).
        They carry headroom, so a captured step graph stays valid while the online updates
        grow the final block (+ceil(L/r) clusters each) until a bound is crossed."""
        need_f, need_c = int(self.led.n_fine.max(initial=0)), int(self.led.n_coarse.max(initial=0))
        if getattr(self, "_bf", None) is None or need_f > self._bf or need_c > self._bc:
            self._bf = min(self.kcap, (need_f + 255) // 128 * 128)
            self._bc = min(self.ccap, (need_c + 255) // 128 * 128) if self.ccap else 0
            self.invalidate_graph()
        return self._bf, self._bc

    def fused_lookup_path(self) -> bool:
        """The flat serving step (bf16 cache and centroids, d = 128, 3 <= G <= 8) runs as ONE launch
        (mpa_decode_step) when its cluster grid fits the device in one wave; hierarchical, fp32
        (parity), d != 128 and oversized (ledgers x centroids) steps use the staged kernels."""
        if not (self.cfg.hierarchy is None and self.dtype == torch.bfloat16 and self.d == 128 and 3 <= self.G <= 8
                and not self.led.lookup_f64):
            return False
        bound = self._cluster_bounds()[0]  # the cluster bound the step is launched with
        if getattr(self, "_fits_for", None) != bound:
            self._fits_for, self._fits = bound, bool(_lib.lib().mpa_decode_step_fits(self.L, self.G, bound))
        return self._fits

    def lookup_step(self, q: torch.Tensor, k_new: torch.Tensor | None = None,
                    v_new: torch.Tensor | None = None) -> None:
        """Flat serving path, ONE launch (mpa_decode_step): both query views (q_rot for the fused
        kernel), fp64 logits, Eq. 1, budgeted selection, the token list and the contiguous-centroid
        weights; with k_new / v_new ([n_seq, Hkv, d] fp32) the step's token is appended after the
        lists were cut (the last CTA advances the device lengths)."""
        self._bound_fine, self._bound_coarse = self._cluster_bounds()
        if int(self.led.n_fine.min()) == 0:
            raise ConfigError("ledger has no clusters")
        qf = q.float().contiguous()
        kf = k_new.float().contiguous() if k_new is not None else None
        vf = v_new.float().contiguous() if v_new is not None else None
        replacement = 0 if self.mode == "flat-no-replacement" else 1
        call("mpa_decode_step", ptr(qf), ptr(kf), ptr(vf), self.cache_struct, ptr(self.cs_lk), ptr(self.inv_freq),
             self.Hkv, self.G, self.led.fine_level(), ptr(self.budget), ptr(self.sink_end_d),
             ptr(self.buffer_start_d), ptr(self.cache_len_d), ptr(self.ntok_dense_d), ptr(self.append_ticket),
             replacement, ptr(self.flag), ptr(self.sel_tokens), ptr(self.tok), self.tok_cap, ptr(self.stats),
             self._bound_fine, ptr(self.q_rot), ptr(self.rej_w) if replacement else None, self.rej_cap, stream_ptr())

    def _contiguous_ok(self) -> bool:
        """Flat level, bf16 centroids, d = 128, G <= 8: the fused decode kernel takes the
        contiguous-centroid list (every fine centroid in order, the selected ones weighted -inf)."""
        return (self.cfg.hierarchy is None and self.dtype == torch.bfloat16 and self.d == 128 and self.G <= 8
                and not self.led.lookup_f64)

    def lookup(self, q: torch.Tensor, staged: bool = False) -> None:
        """K9 + K10 + work lists (flat or hierarchical) for the fp32 queries q [n_seq, Hq, d].  On the
        flat serving path this is the single-launch decode step (the output included) unless
        `staged` asks for the separate logits / selection kernels (the same lists; the path every
        step takes when the single launch does not fit the device)."""
        st = stream_ptr()
        self._bound_fine, self._bound_coarse = self._cluster_bounds()
        G, L = self.G, self.L
        fine = self.led.fine_level()
        replacement = 0 if self.mode == "flat-no-replacement" else 1
        if self.cfg.hierarchy is None and int(self.led.n_fine.min()) == 0:
            raise ConfigError("ledger has no clusters")
        if self.fused_lookup_path() and not staged:  # one launch (the exact view included)
            self.lookup_step(q)
            return
        self.rotate(q, exact=False, lookup=True)
        tiled = self.d in (64, 128)
        cs = self.cstats if tiled else None
        # e^(l - chunk max) from the logits kernel (bf16 serving centroids only)
        el = self.elocal if (tiled and not self.led.lookup_f64) else None
        if self.cfg.hierarchy is None:
            # contiguous-centroid list: the logits kernel writes every centroid's replacement weight
            # (no fp64 logits array), the selection masks the selected ones (no rejected list)
            contig = self._contiguous_ok()
            lg = None if contig else self.logits
            call("mpa_centroid_logits", ptr(self.q_lk), self.Hkv, G, self.d, fine, None,
                 None, self.kcap, ptr(lg), ptr(cs), ptr(el), self._bound_fine, ptr(self.rej_w) if contig else None,
                 self.rej_cap, None, None, st)
            call("mpa_select_worklist", fine, None, G, ptr(lg), ptr(el), None, None, self.kcap, ptr(cs),
                 None, None,
                 ptr(self.budget), ptr(self.sink_end_d), ptr(self.buffer_start_d), ptr(self.cache_len_d), self.Hkv,
                 L, replacement, ptr(self.flag), ptr(self.sel_tokens), ptr(self.tok), self.tok_cap,
                 None if contig else ptr(self.rej), ptr(self.rej_w), self.rej_cap, ptr(self.stats), self._bound_fine,
                 st)
        else:
            if int(self.led.n_coarse.min()) == 0:
                raise ConfigError("ledger has no coarse clusters")
            coarse = self.led.coarse_level()
            ccs = self.ccstats if tiled else None
            cel = self.celocal if el is not None else None
            call("mpa_centroid_logits", ptr(self.q_lk), self.Hkv, G, self.d, coarse, None, None, self.ccap,
                 ptr(self.clogits), ptr(ccs), ptr(cel), self._bound_coarse, None, 0, None, None, st)
            call("mpa_select", ptr(self.clogits), G, None, ptr(self.led.ccount), self.ccap, ptr(self.led.csize),
                 self.ccap, None, None, None, None, 0, ptr(self.cbudget), L, ptr(self.cflag),
                 ptr(self.csel_tokens), ptr(ccs), ptr(cel), self._bound_coarse, st)
            call("mpa_hier_candidates", coarse, ptr(self.cflag), L, ptr(self.cand), ptr(self.n_cand), self.kcap, st)
            call("mpa_centroid_logits", ptr(self.q_lk), self.Hkv, G, self.d, fine, ptr(self.cand), ptr(self.n_cand),
                 self.kcap, ptr(self.logits), ptr(cs), ptr(el), self._bound_fine, None, 0, None, None, st)
            call("mpa_select_worklist", fine, coarse, G, ptr(self.logits), ptr(el), ptr(self.cand), ptr(self.n_cand),
                 self.kcap, ptr(cs), ptr(self.cflag), ptr(self.clogits), ptr(self.budget), ptr(self.sink_end_d),
                 ptr(self.buffer_start_d), ptr(self.cache_len_d), self.Hkv, L, replacement, ptr(self.flag),
                 ptr(self.sel_tokens), ptr(self.tok), self.tok_cap, ptr(self.rej), ptr(self.rej_w), self.rej_cap,
                 ptr(self.stats), self._bound_fine, st)

    def fused(self, n_split: int | None = None) -> torch.Tensor:
        """K11 + K12 over the current work lists.  n_split None / 0: one full wave of the
        stream-K grid (bf16) or automatic splits (fp32); > 0: that many CTAs per ledger."""
        S = int(n_split or 0)
        ws = self._workspace(S)
        st = stream_ptr()
        rej, rej_w, n_rej = self._centroid_terms()
        ckc = self.led.cvc if self.led.hierarchy else None
        call("mpa_sparse_decode", self.cache_struct, ptr(self.q_rot), self.Hkv, self.G, ptr(self.tok),
             ptr(self.stats[0]), self.tok_cap, ptr(rej), ptr(rej_w), ptr(n_rej), self.rej_cap,
             ptr(self.led.vc), self.kcap, ptr(ckc), self.ccap, S, ptr(ws), ws.numel(), ptr(self.out), st)
        return self.out

    def _centroid_terms(self, contiguous: bool | None = None):
        """(rej, rej_w, n_rej) of mpa_sparse_decode: none, the rejected list, or (contiguous: the flat
        bf16 serving path) every fine centroid in order, selected ones weighted -inf."""
        if self.mode == "flat-no-replacement":
            return None, None, None
        if contiguous is None:
            contiguous = self._contiguous_ok()
        if contiguous:
            return None, self.rej_w, self.led.count
        return self.rej, self.rej_w, self.stats[1]

    def attend(self, q: torch.Tensor, n_split: int | None = None) -> torch.Tensor:
        """One multipole decode step over the current cache; q fp32 [n_seq, Hq, d] (device)."""
        if self.mode == "oracle":
            return self.attend_dense(q, n_split)
        if self.fused_lookup_path():
            self.lookup(q)  # the single-launch lookup forms the exact view too
        else:
            self.rotate(q, exact=True, lookup=False)
            self.lookup(q)
        return self.fused(n_split)

    def attend_dense(self, q: torch.Tensor, n_split: int | None = None) -> torch.Tensor:
        """Dense exact attention over [0, cache_len) with the same kernel (K13 comparator)."""
        self.rotate(q)
        S = int(n_split or 0)
        ws = self._workspace(S)
        call("mpa_sparse_decode", self.cache_struct, ptr(self.q_rot), self.Hkv, self.G, None, ptr(self.ntok_dense_d),
             0, None, None, None, 0, None, 0, None, 0, S, ptr(ws), ws.numel(), ptr(self.out), stream_ptr())
        return self.out

    # ------------------------------------------------------------------ pipeline
    def prefill(self) -> None:
        """Index the prompt already written with write_tokens (pipeline.py:69-94)."""
        from . import clustering

        if self.mode == "oracle":
            self.set_prompt_layout()
        elif self.mode == "positional-baseline":
            clustering.prefill_positional(self)
        else:
            clustering.prefill_ledgers(self)
        self.cursor = 0

    def needs_update(self) -> list[int]:
        if self.mode == "oracle":
            return []
        L = self.cfg.local_buffer
        return np.flatnonzero(self.cache_len - self.buffer_start >= 2 * L).tolist()

    # ------------------------------------------------------------------ CUDA graph of a step
    def _graphable(self) -> bool:
        return self.use_graphs and self.mode in ("multipole", "flat-no-replacement")

    def invalidate_graph(self) -> None:
        """The captured step bakes in ledger-dependent launch arguments (cluster counts, split
        sizes): any change to the ledgers or the layout drops it."""
        self._graph = None

    def _capture_step(self) -> None:
        self.n_captures += 1
        n, Hq, Hkv, d, dev = self.n_seq, self.Hq, self.Hkv, self.d, self.device
        # the graph's inputs as one block (q, k, v back to back): mpa_step_host fills it from host
        nq, nk = n * Hq * d, n * Hkv * d
        self._gin = torch.zeros(nq + 2 * nk, dtype=torch.float32, device=dev)
        self._gq = self._gin[:nq].view(n, Hq, d)
        self._gk = self._gin[nq:nq + nk].view(n, Hkv, 1, d)
        self._gv = self._gin[nq + nk:].view(n, Hkv, 1, d)
        self._workspace(0)
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.attend(self._gq)  # warm-up outside the capture (function attributes, tensor maps)
        torch.cuda.current_stream().wait_stream(side)
        self._fev = ((torch.cuda.Event(enable_timing=True, external=True),
                      torch.cuda.Event(enable_timing=True, external=True)) if self.time_fused else None)
        self._bound = None  # the step kernel reads the graph's own input buffers
        self._graph_raw = None
        if self.fused_lookup_path():
            # two launches: lookup + both query views + the append (mpa_decode_step), fused decode;
            # the graph is kept so that its step kernel can be pointed at the caller's q / k / v
            g = torch.cuda.CUDAGraph(keep_graph=True)
            with torch.cuda.graph(g):
                self.lookup_step(self._gq, self._gk[:, :, 0], self._gv[:, :, 0])
                if self._fev:
                    self._fev[0].record()
                self.fused()
                if self._fev:
                    self._fev[1].record()
            g.instantiate()
            self._graph = g
            self._gexec = self._raw_exec(g)
            try:
                self._graph_raw = int(g.raw_cuda_graph()) or None
            except Exception:
                self._graph_raw = None
            return
        g = torch.cuda.CUDAGraph()
        exact_br, append_br = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        with torch.cuda.graph(g):
            # critical path: q_lk -> logits -> select + work lists -> fused decode.  Off it, on
            # graph branches: the exact-view rotation (needed only by the fused kernel) and the KV
            # append (writes row cache_len, which this step's lists never read; it advances the
            # length counters after the selection has read them)
            main = torch.cuda.current_stream()
            exact_br.wait_stream(main)
            with torch.cuda.stream(exact_br):
                self.rotate(self._gq, exact=True, lookup=False)
            self.lookup(self._gq)  # the lookup-view rotation runs inside the lookup kernel (flat bf16 path)
            append_br.wait_stream(main)
            # the exact-view rotation reads cache_len_d, which the append advances: order them
            append_br.wait_stream(exact_br)
            with torch.cuda.stream(append_br):
                call("mpa_kv_append", self.cache_struct, ptr(self._gk), ptr(self._gv), self.Hkv, 1,
                     ptr(self.cache_len_d), ptr(self.ntok_dense_d), ptr(self.inv_freq), ptr(self.append_ticket),
                     stream_ptr())
            main.wait_stream(exact_br)
            if self._fev:
                self._fev[0].record()
            self.fused()
            if self._fev:
                self._fev[1].record()
            main.wait_stream(append_br)
        self._graph = g
        self._gexec = self._raw_exec(g)

    def _bind_inputs(self, q=None, k=None, v=None) -> None:
        """Point the captured step kernel at (q, k, v), or back at the graph's own input buffers."""
        key = None if q is None else (q.data_ptr(), k.data_ptr(), v.data_ptr())
        if key != self._bound:
            if q is None:
                q, k, v = self._gq, self._gk, self._gv
            call("mpa_decode_step_rebind", self._graph_raw, self._gexec, ptr(q), ptr(k), ptr(v))
            self._bound = key

    @staticmethod
    def _raw_exec(g) -> int | None:
        """The cudaGraphExec_t of a captured step, for mpa_step_host (None: torch does not expose it)."""
        try:
            return int(g.raw_cuda_graph_exec()) or None
        except Exception:
            return None

    def step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor) -> torch.Tensor:
        """Attend, append the step's token, then run the online update when a buffer holds 2L
        tokens (pipeline.py:124-191).  q [n_seq, Hq, d], k_new / v_new [n_seq, Hkv, d] (fp32).
        Between ledger changes the attend + append chain replays as one CUDA graph."""
        return self._step(q, k_new, v_new, host=False)

    def _step(self, q, k_new, v_new, host: bool) -> torch.Tensor:
        if self._graphable():
            self.reserve(1)
            self._cluster_bounds()  # recaptures only if the cluster counts outgrew the captured bounds
            if self._graph is None:
                self._capture_step()
            direct = (not host and self._graph_raw is not None and self._gexec is not None
                      and all(x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.data_ptr() % 16 == 0
                              for x in (q, k_new, v_new))
                      and q.numel() == self._gq.numel() and k_new.numel() == self._gk.numel()
                      and v_new.numel() == self._gv.numel())
            if direct:  # the step kernel reads the caller's tensors: no staging copy
                self._bind_inputs(q, k_new, v_new)
            else:
                if self._graph_raw is not None:
                    self._bind_inputs()
                if host:  # host -> device straight into the graph's input buffers
                    self._gq.copy_(q, non_blocking=True)
                    self._gk.copy_(k_new[:, :, None], non_blocking=True)
                    self._gv.copy_(v_new[:, :, None], non_blocking=True)
                elif all(x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.numel() % 4 == 0
                         and x.data_ptr() % 16 == 0 for x in (q, k_new, v_new)):
                    # one launch stages q, k, v into the graph's input buffers
                    call("mpa_stage3", ptr(self._gq), ptr(q), q.numel(), ptr(self._gk), ptr(k_new),
                         k_new.numel(), ptr(self._gv), ptr(v_new), v_new.numel(), stream_ptr())
                else:
                    self._gq.copy_(q)
                    self._gk.copy_(k_new[:, :, None])
                    self._gv.copy_(v_new[:, :, None])
            self._graph.replay()
            self.cache_len += 1
            out = self.out
        else:
            if host:
                q, k_new, v_new = (x.to(self.device, non_blocking=True) for x in (q, k_new, v_new))
            if self.fused_lookup_path() and self.mode != "oracle":
                self.reserve(1)
                self.lookup_step(q, k_new, v_new)
                out = self.fused()
                self.cache_len += 1
            else:
                out = self.attend(q)
                self.write_tokens(k_new[:, :, None], v_new[:, :, None])
        self._post_step()
        return out

    def _post_step(self) -> None:
        from . import clustering

        todo = self.needs_update()
        self.last_update = None
        if todo:
            if self.mode == "positional-baseline":
                self.last_update = clustering.positional_update(self, todo)
            else:
                self.last_update = clustering.online_update(self, todo, self.cursor)
            # the captured graph's launch arguments stay valid while the cluster bounds hold
            self._cluster_bounds()
        self.cursor += 1

    def step_host(self, q_host: torch.Tensor, k_host: torch.Tensor, v_host: torch.Tensor,
                  out_host: torch.Tensor) -> torch.Tensor:
        """Public end-to-end step from HOST buffers (pinned for overlap): copies q / k / v in,
        runs `step`, copies the output back into out_host; all on the current stream."""
        if self._graphable() and all(not x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
                                     for x in (q_host, k_host, v_host, out_host)):
            self.reserve(1)
            self._cluster_bounds()
            if self._graph is None:
                self._capture_step()
            if self._gexec is not None and q_host.numel() == self._gq.numel() and \
                    k_host.numel() == self._gk.numel() and v_host.numel() == self._gv.numel() and \
                    out_host.numel() == self.out.numel() and self.out.dtype == torch.float32:
                # copies in, the step graph, the copy out: one native call
                if self._graph_raw is not None:
                    self._bind_inputs()
                call("mpa_step_host", self._gexec, ptr(self._gin), ptr(q_host), q_host.numel() * 4, ptr(k_host),
                     k_host.numel() * 4, ptr(v_host), v_host.numel() * 4, ptr(out_host), ptr(self.out),
                     out_host.numel() * 4, torch._C._cuda_getCurrentRawStream(self._dev_idx))
                self.cache_len += 1
                self._post_step()
                return out_host
        out = self._step(q_host, k_host, v_host, host=True)
        out_host.copy_(out, non_blocking=True)
        return out_host

    def last_fused_ms(self) -> float | None:
        """Device time of the fused kernel inside the last graph replay (time_fused = True;
        call after synchronising)."""
        return self._fev[0].elapsed_time(self._fev[1]) if self._fev else None

    def export_ledger(self, l: int) -> HostLedger:
        s = l // self.Hkv
        return self.led.export(l, int(self.sink_end[s]), int(self.buffer_start[s]), int(self.cache_len[s]),
                               int(self.splits[l]))

    def head_stats(self) -> np.ndarray:
        """[L, 4]: n_tok, n_rej, selected tokens, selected clusters (host copy)."""
        return self.stats.cpu().numpy().T
