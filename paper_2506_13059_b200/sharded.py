"""Sequence-sharded decode: one long context spread over P ranks (BASELINE config 5).

Every ledger's sealed W-blocks are split contiguously over the ranks; the last rank also owns
the final block, the sinks and the local buffer, so the online update stays rank-local.  Cluster
ids are global (gid_off[l] + local id) and blocks are assigned in order, so the reference's
(block, cluster) tie-break order survives the split.  A decode step exchanges three small
messages, one all-gather each (include/mpattn.h, "Sequence-sharded decode"):

  1. per (ledger, q-head) (M, Z) of Eq. 1 -> global normalisers (attention.py:276-278);
  2. each rank's candidates that can be globally selected (its local take-while-cum<B prefix,
     <= B + 1 entries, and their count, in one message) -> the same global crossing candidate on
     every rank (attention.py:192-207);
  3. per (ledger, q-head) unnormalised (m, s, a) partials -> LSE merge (attention.py:230-239).

`Comm` abstracts the all-gather: `TorchComm` uses torch.distributed (NCCL on the GPU tensors
in a `torchrun` job; gloo works for CPU tensors), `LocalGroup` emulates P ranks inside one
process (lock-step phases) so the sharded algorithm is testable on one GPU.  Heads and batch
shard without any exchange (bench.py replicas).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import MpaCache, call, dtype_code, ptr, stream_ptr
from .core import ConfigError, EngineConfig, HeadLayout
from .engine import DecodeEngine

PREFIX_ENTRY_BYTES = 16  # mpa_prefix_entry
CROSS_BYTES = 16         # mpa_cross


def owned_blocks(rank: int, world: int):
    """Block filter of `rank`: sealed blocks split contiguously (lower ranks first), the final
    block (index n_blocks - 1) on the last rank."""

    def owned(b: int, n_blocks: int) -> bool:
        n_sealed = n_blocks - 1
        if b == n_blocks - 1:
            return rank == world - 1
        lo = n_sealed * rank // world
        hi = n_sealed * (rank + 1) // world
        return lo <= b < hi

    return owned


class TorchComm:
    """All-gather over torch.distributed (NCCL for CUDA tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        t = t.contiguous()
        if self.dist.get_backend(self.group) == "nccl":
            out = torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t.reshape(-1), group=self.group)
            return out.view((self.world,) + tuple(t.shape))
        # gloo: host tensors (a CUDA tensor makes the round trip through host memory)
        src = t.cpu() if t.is_cuda else t
        parts = [torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(parts, src, group=self.group)
        return torch.stack(parts).to(t.device)


class ShardedDecodeEngine:
    """One rank's share of a sequence-sharded decode layer (flat 1-level clustering)."""

    def __init__(self, cfg: EngineConfig, layout: HeadLayout, n_seq: int, tcap: int, rank: int, world: int,
                 dtype: torch.dtype = torch.bfloat16, device="cuda"):
        if cfg.hierarchy is not None:
            raise ConfigError("sequence-sharded decode supports the flat (1-level) index")
        self.rank, self.world = rank, world
        self.eng = DecodeEngine(cfg, layout, n_seq, tcap=tcap, dtype=dtype, device=device, use_graphs=False)
        e = self.eng
        L, G, d, dev = e.L, e.G, e.d, e.device
        self.tail = rank == world - 1
        self.prefix_cap = cfg.token_budget + 1
        self.mz_loc = torch.zeros(L, G, 2, dtype=torch.float64, device=dev)
        self.mz = torch.zeros(L, G, 2, dtype=torch.float64, device=dev)
        # one message for exchange 2: the candidate prefixes [L, cap] entries then their counts [L]
        pb = L * self.prefix_cap * PREFIX_ENTRY_BYTES
        self.msg = torch.zeros(pb + 4 * L, dtype=torch.uint8, device=dev)
        self.prefix = self.msg[:pb].view(L, self.prefix_cap * PREFIX_ENTRY_BYTES)
        self.prefix_n = self.msg[pb:].view(torch.int32)
        self.cross = torch.zeros(L, CROSS_BYTES, dtype=torch.uint8, device=dev)
        self.part = torch.zeros(L, G, d + 2, dtype=torch.float32, device=dev)
        self.gid_off = torch.zeros(L, dtype=torch.int32, device=dev)
        self.zero_sinks = torch.zeros(n_seq, dtype=torch.int32, device=dev)

    # ------------------------------------------------------------------ setup
    def write_tokens(self, k: torch.Tensor, v: torch.Tensor) -> None:
        self.eng.write_tokens(k, v)

    def prefill_local(self) -> None:
        from . import clustering

        clustering.prefill_ledgers(self.eng, owned=owned_blocks(self.rank, self.world))

    def set_gid_offsets(self, n_fine_all: np.ndarray) -> None:
        """n_fine_all [P, L]: every rank's local cluster count per ledger."""
        off = np.asarray(n_fine_all, np.int64)[: self.rank].sum(axis=0) if self.rank else np.zeros(self.eng.L)
        self.gid_off.copy_(torch.as_tensor(off, dtype=torch.int32))

    def _layout(self):
        e = self.eng
        if self.tail:
            return e.sink_end_d, e.buffer_start_d
        # no sinks / buffer on the other ranks: buffer_start = cache_len -> empty buffer
        return self.zero_sinks, e.cache_len_d

    def _contiguous(self) -> bool:
        """Flat bf16 d=128 ledgers: the logits kernel writes every centroid's replacement weight and
        the fused kernel streams the value centroids in order (selected ones weighted -inf)."""
        e = self.eng
        return e.fused_lookup_path() and not e.led.lookup_f64 and e.mode == "multipole"

    # ------------------------------------------------------------------ decode phases
    def phase_norms(self, q: torch.Tensor) -> torch.Tensor:
        """Rotate q, local logits; returns this rank's (M, Z) [L, G, 2]."""
        e = self.eng
        if int(e.led.n_fine.min()) == 0:
            raise ConfigError("ledger has no clusters on this rank")
        e.rotate(q)
        st = stream_ptr()
        fine = e.led.fine_level()
        el = e.elocal if not e.led.lookup_f64 else None
        dense = self._contiguous()
        call("mpa_centroid_logits", ptr(e.q_lk), e.Hkv, e.G, e.d, fine, None, None, e.kcap, ptr(e.logits),
             ptr(e.cstats), ptr(el), int(e.led.n_fine.max()), ptr(e.rej_w) if dense else None, e.rej_cap, None, None,
             st)
        call("mpa_head_norms", ptr(e.cstats), e.cstats.shape[1], ptr(e.led.count), e.L, e.G, ptr(self.mz_loc), st)
        return self.mz_loc

    def phase_prefix(self, mz_all: torch.Tensor) -> torch.Tensor:
        """Global normalisers from every rank's (M, Z); this rank's candidate prefix and its counts in
        one message (self.msg)."""
        e = self.eng
        st = stream_ptr()
        call("mpa_merge_norms", ptr(mz_all), self.world, e.L, e.G, ptr(self.mz), st)
        self.prefix_n.zero_()
        sink, buf = self._layout()
        el = e.elocal if not e.led.lookup_f64 else None
        call("mpa_select_worklist_sharded", e.led.fine_level(), e.G, ptr(e.logits), ptr(el), ptr(e.cstats),
             ptr(e.budget), ptr(sink), ptr(buf), ptr(e.cache_len_d), e.Hkv, 1, ptr(e.flag), ptr(e.sel_tokens),
             ptr(e.tok), e.tok_cap, ptr(e.rej), ptr(e.rej_w), e.rej_cap, ptr(e.stats), int(e.led.n_fine.max()),
             ptr(self.mz), None, ptr(self.prefix), ptr(self.prefix_n), self.prefix_cap, ptr(self.gid_off), st)
        return self.msg

    def split_msgs(self, msg_all: torch.Tensor):
        """[P, msg] -> (prefixes [P, L, cap] entries, counts [P, L]) as the contiguous arrays
        mpa_global_cut reads."""
        e = self.eng
        pb = e.L * self.prefix_cap * PREFIX_ENTRY_BYTES
        return msg_all[:, :pb].contiguous(), msg_all[:, pb:].contiguous().view(torch.int32)

    def phase_partials(self, prefix_all: torch.Tensor, prefix_n_all: torch.Tensor) -> torch.Tensor:
        """Global crossing candidate, local work lists, local fused attention -> partials."""
        e = self.eng
        st = stream_ptr()
        call("mpa_global_cut", ptr(prefix_all), ptr(prefix_n_all), self.world, e.L, self.prefix_cap, ptr(e.budget),
             ptr(self.cross), st)
        rej = e._centroid_terms(self._contiguous())[0] if e.mode != "flat-no-replacement" else e.rej
        sink, buf = self._layout()
        el = e.elocal if not e.led.lookup_f64 else None
        call("mpa_select_worklist_sharded", e.led.fine_level(), e.G, ptr(e.logits), ptr(el), ptr(e.cstats),
             ptr(e.budget), ptr(sink), ptr(buf), ptr(e.cache_len_d), e.Hkv, 1, ptr(e.flag), ptr(e.sel_tokens),
             ptr(e.tok), e.tok_cap, ptr(rej), ptr(e.rej_w), e.rej_cap, ptr(e.stats), int(e.led.n_fine.max()),
             ptr(self.mz), ptr(self.cross), None, None, self.prefix_cap, ptr(self.gid_off), st)
        ws = e._workspace(0)
        rej, rej_w, n_rej = e._centroid_terms(self._contiguous())
        call("mpa_sparse_decode_partials", e.cache_struct, ptr(e.q_rot), e.Hkv, e.G, ptr(e.tok), ptr(e.stats[0]),
             e.tok_cap, ptr(rej), ptr(rej_w), ptr(n_rej), e.rej_cap, ptr(e.led.vc), e.kcap, None, 0, 0,
             ptr(ws), ws.numel(), ptr(self.part), st)
        return self.part

    def phase_merge(self, parts_all: torch.Tensor) -> torch.Tensor:
        e = self.eng
        call("mpa_merge_rank_partials", ptr(parts_all), self.world, e.L, e.G, e.d, ptr(e.out), stream_ptr())
        return e.out

    def attend(self, q: torch.Tensor, comm) -> torch.Tensor:
        """One sharded decode step on this rank: three all-gathers through `comm` -- (M, Z), the
        candidate-prefix message, the (m, s, a) partials."""
        mz_all = comm.all_gather(self.phase_norms(q))
        prefix_all, prefix_n_all = self.split_msgs(comm.all_gather(self.phase_prefix(mz_all)))
        parts = self.phase_partials(prefix_all, prefix_n_all)
        return self.phase_merge(comm.all_gather(parts))

    def capture_attend(self, q: torch.Tensor, comm) -> None:
        """Capture one whole sharded decode step -- the local kernels AND the three NCCL all-gathers
        -- as one CUDA graph (NCCL collectives are graph-capturable); `attend_graphed` then replays it.
        Valid while this rank's ledgers keep their cluster counts (an online update re-captures)."""
        e = self.eng
        if int(e.led.n_fine.min()) == 0:
            raise ConfigError("ledger has no clusters on this rank")
        self._gq = q.detach().clone()
        e._workspace(0)
        for _ in range(2):  # communicator and allocator warm-up outside the capture
            self.attend(self._gq, comm)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = self.attend(self._gq, comm)
        self._graph, self._gout = g, out
        self._graph_key = e.led.n_fine.copy()

    def attend_graphed(self, q: torch.Tensor, comm) -> torch.Tensor:
        e = self.eng
        if getattr(self, "_graph", None) is None or not np.array_equal(self._graph_key, e.led.n_fine):
            self.capture_attend(q, comm)
        self._gq.copy_(q)
        self._graph.replay()
        return self._gout

    def step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, comm) -> torch.Tensor:
        """attend, append the step's token on every rank (pipeline.py:137-159), and run the online
        update on the tail rank, which owns the final block, the sinks and the buffer (the update is
        rank-local: clustering.py:404-472).  A split seals the block on the tail rank; cluster ids stay
        global because the tail is the last rank."""
        from . import clustering

        e = self.eng
        out = self.attend(q, comm)
        e.write_tokens(k_new[:, :, None], v_new[:, :, None])
        if self.tail:
            todo = e.needs_update()
            if todo:
                clustering.online_update(e, todo, e.cursor)
        e.cursor += 1
        return out


class LocalGroup:
    """P sharded engines in one process, advanced phase by phase (the all-gathers become
    concatenations) -- the single-GPU check that sharded == unsharded."""

    def __init__(self, engines: list[ShardedDecodeEngine]):
        self.engines = engines

    def prefill(self) -> None:
        for e in self.engines:
            e.prefill_local()
        n_all = np.stack([e.eng.led.n_fine for e in self.engines])
        for e in self.engines:
            e.set_gid_offsets(n_all)

    def attend(self, q: torch.Tensor) -> torch.Tensor:
        mz_all = torch.stack([e.phase_norms(q).clone() for e in self.engines])
        msg_all = torch.stack([e.phase_prefix(mz_all).clone() for e in self.engines])
        prefix_all, prefix_n_all = self.engines[0].split_msgs(msg_all)
        parts_all = torch.stack([e.phase_partials(prefix_all, prefix_n_all).clone() for e in self.engines])
        outs = [e.phase_merge(parts_all).clone() for e in self.engines]
        return outs[0]
