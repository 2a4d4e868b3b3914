"""Reference-compatible prefill / step / run on the B200 engine (drop-in for
pkg/src/multipole_attn/pipeline.py:23-220).

Same signatures, modes, cadence and exceptions as the reference:
  * `prefill(trace, cfg, mode)` builds the per-kv-head ledgers on the GPU,
  * `step(state, queries, new_keys, new_values, oracle, audit, timers)` attends BEFORE appending
    the step's token and runs the online update when the buffer reaches 2L,
  * outputs are float64 (Hq, d) numpy arrays and a `DecodeReport` per step.
Extra keyword `dtype`: float64 (default) keeps the reference's numerics -- the ledgers come from the
engine's clustering kernels and every attention partial runs on the fp64 kernels behind the
module-level API (attention.decode_step_attention, csrc/mpa_refapi.cu); float32 / bfloat16 run the
batched serving kernels (the single-launch lookup and the stream-K fused decode) on a cache of that
dtype.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from .attention import DecodeReport, StepHeadResult, oracle_topk_tokens
from .core import ConfigError, EngineConfig, KvTrace
from .engine import DecodeEngine
from .rope import RopeParams

MODES = ("multipole", "oracle", "flat-no-replacement", "positional-baseline")


@dataclass
class EngineState:
    trace: KvTrace
    cfg: EngineConfig
    mode: str
    engine: DecodeEngine
    cursor: int = 0

    @property
    def cache_len(self) -> int:
        return self.trace.prompt_len + self.cursor

    fp64: bool = False
    _ref_ledgers: list | None = None

    @property
    def ledgers(self):
        """The device ledgers as reference BlockLedger objects (one per kv-head; pipeline.py:55-62)."""
        if self.mode == "oracle":
            return []
        from .clustering import _to_block_ledger

        if self._ref_ledgers is None:
            self._ref_ledgers = [_to_block_ledger(self.engine, h) for h in range(self.trace.layout.num_kv_heads)]
        return self._ref_ledgers

    @property
    def stores(self):
        """Per-kv-head views of the device KV cache (pipeline.py:26-52 `_KvStore`: n, keys, values)."""
        return [_KvStoreView(self.engine, h) for h in range(self.trace.layout.num_kv_heads)]


class _KvStoreView:
    """Read-only view of one kv-head's cached (pre-rotation) keys and values."""

    def __init__(self, eng: DecodeEngine, h: int):
        self._eng, self._h = eng, h

    @property
    def n(self) -> int:
        return int(self._eng.cache_len[0])

    @property
    def keys(self) -> np.ndarray:
        return self._eng.k_raw[self._h, : self.n].float().cpu().numpy()

    @property
    def values(self) -> np.ndarray:
        return self._eng.values(self._h, torch.arange(self.n)).float().cpu().numpy()


def prefill(trace: KvTrace, cfg: EngineConfig, mode: str = "multipole", dtype: torch.dtype = torch.float64,
            capacity: int | None = None) -> EngineState:
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    lay = trace.layout
    P = trace.prompt_len
    if P <= cfg.sink_tokens and mode != "oracle":
        raise ConfigError(f"prompt_len {P} must exceed sink_tokens {cfg.sink_tokens}")
    fp64 = dtype == torch.float64
    eng = DecodeEngine(cfg, lay, 1, tcap=capacity or max(16, trace.total_len + 1),
                       dtype=torch.float32 if fp64 else dtype, mode=mode)
    dev = eng.device
    eng.write_tokens(torch.as_tensor(trace.keys[:, :P], device=dev)[None],
                     torch.as_tensor(trace.values[:, :P], device=dev)[None])
    eng.prefill()
    return EngineState(trace=trace, cfg=cfg, mode=mode, engine=eng, fp64=fp64)


def _refs(eng: DecodeEngine, h: int, flag: np.ndarray, cand: np.ndarray | None) -> list:
    """(block, cluster, 2) refs of the selected fine clusters of kv-head h (sorted by ref), from host
    copies of the selection flags (and, hierarchy, the candidate lists)."""
    led = eng.led
    if eng.cfg.hierarchy is None:
        ids = np.flatnonzero(flag[: int(led.n_fine[h])])
    else:
        n = int(eng.n_cand[h]) if cand is None else cand.size
        ids = np.sort(cand[flag[:n] == 1])
    rows = led.blocks[h]
    if not rows or ids.size == 0:
        return []
    f0 = np.fromiter((row.f0 for row in rows), np.int64, len(rows))
    fk = np.fromiter((row.fk for row in rows), np.int64, len(rows))
    bi = np.searchsorted(f0, ids, side="right") - 1  # block of each selected fine id (blocks ascend)
    keep = (bi >= 0) & (ids < f0[np.maximum(bi, 0)] + fk[np.maximum(bi, 0)])
    bi, loc = bi[keep], ids[keep] - f0[bi[keep]]
    return list(zip(bi.tolist(), loc.tolist(), [2] * int(bi.size)))


def _attend_fp64(state: EngineState, queries, oracle: bool, timers):
    """The reference's numerics: attention.decode_step_attention over the engine's ledgers and cache,
    every partial on the fp64 kernels (pipeline.py:137-150); oracle mode: exact attention per q-head
    (pipeline.py:97-121)."""
    from . import attention

    eng, lay, cfg = state.engine, state.trace.layout, state.cfg
    n = int(eng.cache_len[0])
    keys = eng.k_raw[:, :n].double().cpu().numpy()
    values = torch.stack([eng.values(l, torch.arange(n)) for l in range(eng.L)]).double().cpu().numpy()
    q = np.asarray(queries)
    if state.mode == "oracle":
        params = RopeParams(head_dim=lay.head_dim, theta=cfg.rope_theta, window_offset=cfg.window_offset)
        pos = np.arange(n, dtype=np.int64)
        out = np.empty((lay.num_q_heads, lay.head_dim))
        for h in range(lay.num_kv_heads):
            for g in lay.q_heads_of(h):
                out[g] = attention.exact_attention(q[g], n, keys[h], values[h], pos, params)
        rep = DecodeReport(step=state.cursor, errors=[0.0] * lay.num_q_heads, per_head=[], cache_len=n,
                           sink_count=0, buffer_len=0, num_kv_heads=lay.num_kv_heads, mode="oracle")
        return out, rep
    return attention.decode_step_attention(q, state.ledgers, list(keys), list(values), n, state.cursor, cfg, lay,
                                           mode=state.mode, oracle=oracle, timers=timers)


def _attend_engine(state: EngineState, queries, oracle: bool):
    """The batched serving kernels (bf16 / fp32 cache): one lookup launch (flat) or the staged lookup
    kernels (hierarchy), the fused decode kernel; the report from one batched device -> host copy."""
    eng, lay = state.engine, state.trace.layout
    dev = eng.device
    q = torch.as_tensor(np.asarray(queries, np.float32), device=dev)[None]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    n = int(eng.cache_len[0])
    ev[0].record()
    if state.mode == "oracle":
        out_t = eng.attend_dense(q)
        ev[1].record()
    else:
        if not eng.fused_lookup_path():  # the single-launch lookup forms the exact view itself
            eng.rotate(q, exact=True, lookup=False)
        eng.lookup(q)
        ev[1].record()
        out_t = eng.fused()
    ev[2].record()
    H = lay.num_kv_heads
    flat = state.mode != "oracle" and eng.cfg.hierarchy is None
    # one batched device -> host read (pinned, non-blocking) of everything the report needs: the
    # output, the per-head counters, the token lists (bounded by sinks + buffer + budget + the largest
    # cluster, which every list fits) and the selection flags
    kf = max(int(eng.led.n_fine[:H].max(initial=0)), 1)
    tb = min(eng.tok_cap, int(eng.sink_end[0]) + (n - int(eng.buffer_start[0])) + eng.cfg.token_budget
             + int(eng.led.max_size[:H].max(initial=0)) + 16)
    hb = state.__dict__.setdefault("_host", {})
    def pinned(name, shape, dtype):
        t = hb.get(name)
        if t is None or t.shape != torch.Size(shape) or t.dtype != dtype:
            t = hb[name] = torch.empty(shape, dtype=dtype, pin_memory=True)
        return t
    out_h = pinned("out", (lay.num_q_heads, lay.head_dim), torch.float32)
    out_h.copy_(out_t[0], non_blocking=True)
    if state.mode != "oracle":
        st_h = pinned("stats", (4, H), torch.int32)
        st_h.copy_(eng.stats[:, :H], non_blocking=True)
        tok_h = pinned("tok", (H, tb), torch.int32)
        tok_h.copy_(eng.tok[:H, :tb], non_blocking=True)
        if flat:
            fl_h = pinned("flag", (H, kf), torch.uint8)
            fl_h.copy_(eng.flag[:H, :kf], non_blocking=True)
    torch.cuda.current_stream().synchronize()
    out = out_h.numpy().astype(np.float64)
    errors = topk = None
    if oracle:
        ref = eng.attend_dense(q)[0].double().cpu().numpy()
        errors = list(np.linalg.norm(out - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-300))
    per_head, sel = [], []
    if state.mode != "oracle":
        st = st_h.numpy().T
        ntok = int(st[:H, 0].max())
        if ntok > tb:  # cannot happen (tb bounds every list); read the rest if it did
            tok = eng.tok[:H, :ntok].cpu().numpy()
        else:
            tok = tok_h.numpy()
        flags = fl_h.numpy() if flat else eng.flag[:H, :kf].cpu().numpy()
        cands = None
        if eng.cfg.hierarchy is not None:
            nc = eng.n_cand[:H].cpu().numpy()
            cm = eng.cand[:H, :max(int(nc.max()), 1)].cpu().numpy()
            cands = [cm[h, : int(nc[h])] for h in range(H)]
        ns = min(int(eng.sink_end[0]), n)
        nb = n - int(eng.buffer_start[0])
        for h in range(H):
            sel.append(np.sort(tok[h, ns + nb: st[h, 0]].astype(np.int64)))
            scored = int(eng.led.n_fine[h]) if eng.cfg.hierarchy is None else \
                int(eng.led.n_coarse[h]) + int(cands[h].size)
            per_head.append(StepHeadResult(_refs(eng, h, flags[h], cands[h] if cands else None), int(st[h, 2]),
                                           scored, int(st[h, 1]) if state.mode != "flat-no-replacement" else 0))
    if oracle and state.mode != "oracle":
        # attention.py:500-529: the true top tokens (group-summed exact weight) among the clustered ones,
        # k = the selected token count of the head (budget when none)
        params = RopeParams(head_dim=lay.head_dim, theta=state.cfg.rope_theta, window_offset=state.cfg.window_offset)
        qn = np.asarray(queries, np.float64)
        keys = eng.k_raw[:, :n].double().cpu().numpy()  # the cached (pre-rotation) keys
        topk = [oracle_topk_tokens(qn, list(lay.q_heads_of(h)), keys[h], n, np.arange(min(int(eng.sink_end[0]), n)),
                                   np.arange(int(eng.buffer_start[0]), n), int(sel[h].size), state.cfg.token_budget,
                                   params) for h in range(lay.num_kv_heads)]
    elif oracle:
        topk = [np.zeros(0, np.int64) for _ in range(lay.num_kv_heads)]
    rep = DecodeReport(step=state.cursor, errors=errors if oracle else ([0.0] * lay.num_q_heads
                                                                      if state.mode == "oracle" else None),
                       per_head=per_head, cache_len=n,
                       sink_count=0 if state.mode == "oracle" else min(state.cfg.sink_tokens, n),
                       buffer_len=0 if state.mode == "oracle" else n - int(eng.buffer_start[0]),
                       num_kv_heads=lay.num_kv_heads, selected_indices=sel if sel else None, oracle_topk=topk,
                       mode=state.mode)
    rep.gpu_times = {"lookup": ev[0].elapsed_time(ev[1]) * 1e-3, "exact": ev[1].elapsed_time(ev[2]) * 1e-3}
    return out, rep


def step(state: EngineState, queries, new_keys, new_values, oracle: bool = False, audit: bool = False,
         timers: dict | None = None):
    """pipeline.py:124-191: attend, then append the step's token and run the buffered cluster update
    once the buffer holds 2L tokens.  Mutates state."""
    eng = state.engine
    lay = state.trace.layout
    dev = eng.device
    if state.fp64:
        out, rep = _attend_fp64(state, queries, oracle, timers)
    else:
        out, rep = _attend_engine(state, queries, oracle)
        if timers is not None:
            timers["lookup"] = timers.get("lookup", 0.0) + rep.gpu_times["lookup"]
            timers["exact"] = timers.get("exact", 0.0) + rep.gpu_times["exact"]
            timers["replace"] = timers.get("replace", 0.0)  # fused into the exact kernel
    # append + online update
    t0 = time.perf_counter()
    kn = torch.as_tensor(np.asarray(new_keys, np.float32), device=dev)[None, :, None]
    vn = torch.as_tensor(np.asarray(new_values, np.float32), device=dev)[None, :, None]
    eng.write_tokens(kn, vn)
    if state._ref_ledgers is not None:
        for led in state._ref_ledgers:
            led.total += 1
    todo = eng.needs_update()
    if todo:
        from . import clustering

        if state.mode == "positional-baseline":
            clustering.positional_update(eng, todo)
        else:
            clustering.online_update(eng, todo, eng.cursor)
        torch.cuda.synchronize()
        state._ref_ledgers = None
        rep.update_occurred = True
        rep.update_wall_time = time.perf_counter() - t0
        if audit:
            from .audit import audit_engine

            audit_engine(eng, check_assignment=state.mode != "positional-baseline")
        if timers is not None:
            timers["update"] = timers.get("update", 0.0) + rep.update_wall_time
    eng.cursor += 1
    state.cursor += 1
    return out, rep


def run(trace: KvTrace, cfg: EngineConfig, mode: str = "multipole", oracle: bool = False, audit: bool = False,
        max_steps: int | None = None, collect_outputs: bool = False, dtype: torch.dtype = torch.float64):
    if trace.decode_steps < 1:
        raise ValueError("trace has no decode steps")
    state = prefill(trace, cfg, mode=mode, dtype=dtype)
    n = trace.decode_steps if max_steps is None else min(max_steps, trace.decode_steps)
    reports = []
    for t in range(n):
        pos = trace.prompt_len + t
        out, rep = step(state, trace.queries[:, t], trace.keys[:, pos], trace.values[:, pos], oracle=oracle,
                        audit=audit)
        if collect_outputs:
            rep.outputs = out
        reports.append(rep)
    return reports
