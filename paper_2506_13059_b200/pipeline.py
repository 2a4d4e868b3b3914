"""Reference-compatible prefill / step / run on the B200 engine (drop-in for
pkg/src/multipole_attn/pipeline.py:23-220).

Same signatures, modes, cadence and exceptions as the reference:
  * `prefill(trace, cfg, mode)` builds the per-kv-head ledgers on the GPU,
  * `step(state, queries, new_keys, new_values, oracle, audit, timers)` attends BEFORE appending
    the step's token and runs the online update when the buffer reaches 2L,
  * outputs are float64 (Hq, d) numpy arrays and a `DecodeReport` per step.
Extra keyword `dtype` selects the KV-cache dtype (float32: the 1e-5 parity mode, the default
here because the reference computes in fp64; bfloat16: the serving layout).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .core import ConfigError, EngineConfig, KvTrace
from .engine import DecodeEngine

MODES = ("multipole", "oracle", "flat-no-replacement", "positional-baseline")


@dataclass
class StepHeadResult:
    selected_refs: list
    selected_tokens: int
    scored_centroids: int
    rejected_centroids: int


@dataclass
class DecodeReport:
    """attention.py:390-407."""

    step: int
    errors: list | None
    per_head: list
    cache_len: int
    sink_count: int
    buffer_len: int
    num_kv_heads: int
    update_occurred: bool = False
    update_wall_time: float = 0.0
    selected_indices: list | None = None
    oracle_topk: list | None = None
    mode: str = "multipole"
    outputs: np.ndarray | None = None
    gpu_times: dict = field(default_factory=dict)

    def mean_error(self) -> float:
        return float(np.mean(self.errors)) if self.errors else float("nan")


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

    @property
    def ledgers(self):
        """Host views of the device ledgers (one per kv-head)."""
        if self.mode == "oracle":
            return []
        return [self.engine.export_ledger(h) for h in range(self.trace.layout.num_kv_heads)]


def prefill(trace: KvTrace, cfg: EngineConfig, mode: str = "multipole", dtype: torch.dtype = torch.float32,
            capacity: int | None = None) -> EngineState:
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    lay = trace.layout
    P = trace.prompt_len
    if P <= cfg.sink_tokens and mode != "oracle":
        raise ConfigError(f"prompt_len {P} must exceed sink_tokens {cfg.sink_tokens}")
    eng = DecodeEngine(cfg, lay, 1, tcap=capacity or max(16, trace.total_len + 1), dtype=dtype, mode=mode)
    dev = eng.device
    eng.write_tokens(torch.as_tensor(trace.keys[:, :P], device=dev)[None],
                     torch.as_tensor(trace.values[:, :P], device=dev)[None])
    eng.prefill()
    return EngineState(trace=trace, cfg=cfg, mode=mode, engine=eng)


def _refs(eng: DecodeEngine, h: int) -> list:
    """(block, cluster, 2) refs of the selected fine clusters of kv-head h (sorted by ref)."""
    led = eng.led
    flag = eng.flag[h].cpu().numpy()
    if eng.cfg.hierarchy is None:
        ids = np.flatnonzero(flag[: int(led.n_fine[h])])
    else:
        n = int(eng.n_cand[h])
        cand = eng.cand[h, :n].cpu().numpy()
        ids = np.sort(cand[flag[:n] == 1])
    out = []
    for r_i, row in enumerate(led.blocks[h]):
        for g in ids[(ids >= row.f0) & (ids < row.f0 + row.fk)]:
            out.append((r_i, int(g - row.f0), 2))
    return out


def step(state: EngineState, queries, new_keys, new_values, oracle: bool = False, audit: bool = False,
         timers: dict | None = None):
    eng = state.engine
    lay = state.trace.layout
    dev = eng.device
    q = torch.as_tensor(np.asarray(queries, np.float32), device=dev)[None]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    n = eng.cache_len[0]
    ev[0].record()
    if state.mode == "oracle":
        out_t = eng.attend_dense(q)
        ev[1].record()
        ev[2].record()
    else:
        if not eng.fused_lookup_path():  # the single-launch lookup forms the exact view itself
            eng.rotate(q, exact=True, lookup=False)
        eng.lookup(q)
        ev[1].record()
        out_t = eng.fused()
        ev[2].record()
    out = out_t[0].double().cpu().numpy()
    errors = None
    if oracle:
        ref = eng.attend_dense(q)[0].double().cpu().numpy()
        errors = list(np.linalg.norm(out - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-300))
    per_head, sel = [], []
    if state.mode != "oracle":
        st = eng.head_stats()
        for h in range(lay.num_kv_heads):
            ns = min(int(eng.sink_end[0]), n)
            nb = n - int(eng.buffer_start[0])
            idx = np.sort(eng.tok[h, ns + nb: st[h, 0]].cpu().numpy().astype(np.int64))
            sel.append(idx)
            scored = int(eng.led.n_fine[h]) if eng.cfg.hierarchy is None else \
                int(eng.led.n_coarse[h]) + int(eng.n_cand[h])
            per_head.append(StepHeadResult(_refs(eng, h), int(st[h, 2]), scored,
                                           int(st[h, 1]) if state.mode != "flat-no-replacement" else 0))
    rep = DecodeReport(step=state.cursor, errors=errors if oracle else ([0.0] * lay.num_q_heads
                                                                      if state.mode == "oracle" else None),
                       per_head=per_head, cache_len=int(n),
                       sink_count=0 if state.mode == "oracle" else min(state.cfg.sink_tokens, int(n)),
                       buffer_len=0 if state.mode == "oracle" else int(n - eng.buffer_start[0]),
                       num_kv_heads=lay.num_kv_heads, selected_indices=sel if sel else None, mode=state.mode)
    # append + online update
    t0 = time.perf_counter()
    kn = torch.as_tensor(np.asarray(new_keys, np.float32), device=dev)[None, :, None]
    vn = torch.as_tensor(np.asarray(new_values, np.float32), device=dev)[None, :, None]
    eng.write_tokens(kn, vn)
    todo = eng.needs_update()
    if todo:
        from . import clustering

        if state.mode == "positional-baseline":
            clustering.positional_update(eng, todo)
        else:
            clustering.online_update(eng, todo, eng.cursor)
        torch.cuda.synchronize()
        rep.update_occurred = True
        rep.update_wall_time = time.perf_counter() - t0
        if audit:
            from .audit import audit_engine

            audit_engine(eng, check_assignment=state.mode != "positional-baseline")
    eng.cursor += 1
    state.cursor += 1
    ev[3].record()
    torch.cuda.synchronize()
    rep.gpu_times = {"lookup": ev[0].elapsed_time(ev[1]) * 1e-3, "exact": ev[1].elapsed_time(ev[2]) * 1e-3}
    if timers is not None:
        timers["lookup"] = timers.get("lookup", 0.0) + rep.gpu_times["lookup"]
        timers["exact"] = timers.get("exact", 0.0) + rep.gpu_times["exact"]
        timers["replace"] = timers.get("replace", 0.0)  # fused into the exact kernel
        if rep.update_occurred:
            timers["update"] = timers.get("update", 0.0) + rep.update_wall_time
    return out, rep


def run(trace: KvTrace, cfg: EngineConfig, mode: str = "multipole", oracle: bool = False, audit: bool = False,
        max_steps: int | None = None, collect_outputs: bool = False, dtype: torch.dtype = torch.float32):
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
