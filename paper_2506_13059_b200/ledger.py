"""Device ledger: the reference's per-kv-head `BlockLedger` (clustering.py:37-77) as
struct-of-arrays in HBM, one row per ledger l = seq * n_kv_heads + kv_head.

Fine level (all blocks of a ledger concatenated in block order, so the flat cluster id is the
reference's (block, cluster) ref order):
    kc, vc        [L, kcap, d]   serving dtype (bf16 / fp32) -- what decode reads
    kc64, vc64    [L, kcap, d]   fp64 master copies (what clustering and audits use)
    size          [L, kcap]      int32
    count         [L]            int32 live clusters
    off           [L, kcap + 1]  int32 CSR offsets into mem (block b's members occupy exactly
                                  its token span, so off is one prefix sum over all clusters)
    mem           [L, tcap]      int32 member token ids, ascending within a cluster
Coarse level (hierarchy on): ckc/cvc/ckc64/cvc64 [L, ccap, d], csize, ccount,
    coff [L, ccap + 1] CSR into child [L, kcap] (fine ids, ascending per coarse cluster).
Per-ledger block table (host mirror, changes only at updates): list of
    (start, end, fine_first, fine_count, coarse_first, coarse_count).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import MPA_F64, MpaLevel, dtype_code, ptr


@dataclass
class BlockRow:
    start: int
    end: int
    f0: int      # first fine cluster (flat id)
    fk: int      # fine clusters in this block
    c0: int = 0  # first coarse cluster
    ck: int = 0


@dataclass
class HostLedger:
    """Plain-array view of one ledger, exchanged with tests/oracle and used for audits."""

    sink_end: int
    buffer_start: int
    total: int
    splits: int
    blocks: list = field(default_factory=list)   # BlockRow
    kc: np.ndarray | None = None                  # (K, d) fp64
    vc: np.ndarray | None = None
    size: np.ndarray | None = None                # (K,)
    mem: np.ndarray | None = None                 # concatenated members
    ckc: np.ndarray | None = None
    cvc: np.ndarray | None = None
    csize: np.ndarray | None = None
    child_off: np.ndarray | None = None
    child: np.ndarray | None = None


class DeviceLedgers:
    def __init__(self, n_ledgers: int, d: int, tcap: int, kcap: int, ccap: int, dtype: torch.dtype,
                 hierarchy: bool, device):
        L = n_ledgers
        self.L, self.d, self.tcap, self.kcap, self.ccap = L, d, tcap, kcap, ccap
        self.dtype, self.hierarchy, self.device = dtype, hierarchy, device
        z = dict(device=device)
        self.kc = torch.zeros(L, kcap, d, dtype=dtype, **z)
        self.vc = torch.zeros(L, kcap, d, dtype=dtype, **z)
        self.kc64 = torch.zeros(L, kcap, d, dtype=torch.float64, **z)
        self.vc64 = torch.zeros(L, kcap, d, dtype=torch.float64, **z)
        self.size = torch.zeros(L, kcap, dtype=torch.int32, **z)
        self.count = torch.zeros(L, dtype=torch.int32, **z)
        self.off = torch.zeros(L, kcap + 1, dtype=torch.int32, **z)
        self.mem = torch.zeros(L, tcap, dtype=torch.int32, **z)
        if hierarchy:
            self.ckc = torch.zeros(L, ccap, d, dtype=dtype, **z)
            self.cvc = torch.zeros(L, ccap, d, dtype=dtype, **z)
            self.ckc64 = torch.zeros(L, ccap, d, dtype=torch.float64, **z)
            self.cvc64 = torch.zeros(L, ccap, d, dtype=torch.float64, **z)
            self.csize = torch.zeros(L, ccap, dtype=torch.int32, **z)
            self.ccount = torch.zeros(L, dtype=torch.int32, **z)
            self.coff = torch.zeros(L, ccap + 1, dtype=torch.int32, **z)
            self.child = torch.zeros(L, kcap, dtype=torch.int32, **z)
        # host mirror of the block tables and counts
        self.blocks: list[list[BlockRow]] = [[] for _ in range(L)]
        self.n_fine = np.zeros(L, np.int64)
        self.n_coarse = np.zeros(L, np.int64)
        self._max_size = np.zeros(L, np.int64)
        self._max_size_dev = None  # a pending device-side refresh (online updates), read on demand

    @property
    def max_size(self) -> np.ndarray:
        """Largest fine cluster per ledger (host); an online update leaves it on the device and the
        first reader pays the copy, so the update itself ends without a device sync."""
        if self._max_size_dev is not None:
            self._max_size[:] = self._max_size_dev.cpu().numpy()
            self._max_size_dev = None
        return self._max_size

    def set_max_size_async(self, dev_values: torch.Tensor) -> None:
        """dev_values: every ledger's value (an older pending refresh is superseded)."""
        self._max_size_dev = dev_values

    # -- C-ABI views ---------------------------------------------------------
    @property
    def lookup_f64(self) -> bool:
        """fp32 caches are the parity mode: the lookup reads the fp64 master centroids (exactly
        the reference's operands); bf16 caches serve bf16 centroids (half the bytes)."""
        return self.dtype == torch.float32

    def fine_level(self) -> MpaLevel:
        kc, code = (self.kc64, MPA_F64) if self.lookup_f64 else (self.kc, dtype_code(self.dtype))
        return MpaLevel(ptr(kc), ptr(self.vc), ptr(self.size), ptr(self.count), ptr(self.off), ptr(self.mem),
                        self.kcap, self.tcap, code, self.L)

    def coarse_level(self) -> MpaLevel | None:
        if not self.hierarchy:
            return None
        kc, code = (self.ckc64, MPA_F64) if self.lookup_f64 else (self.ckc, dtype_code(self.dtype))
        return MpaLevel(ptr(kc), ptr(self.cvc), ptr(self.csize), ptr(self.ccount), ptr(self.coff),
                        ptr(self.child), self.ccap, self.kcap, code, self.L)

    # -- host <-> device -----------------------------------------------------
    def load(self, l: int, h: HostLedger) -> None:
        """Install one ledger from host arrays (used by tests and by the checkpoint loader)."""
        K = int(h.size.size)
        if K > self.kcap:
            raise ValueError(f"ledger {l}: {K} clusters > kcap {self.kcap}")
        dev = self.device
        self.kc64[l, :K] = torch.as_tensor(h.kc, dtype=torch.float64, device=dev)
        self.vc64[l, :K] = torch.as_tensor(h.vc, dtype=torch.float64, device=dev)
        self.kc[l, :K] = self.kc64[l, :K].to(self.dtype)
        self.vc[l, :K] = self.vc64[l, :K].to(self.dtype)
        self.size[l, :K] = torch.as_tensor(h.size, dtype=torch.int32, device=dev)
        self.count[l] = K
        off = np.zeros(K + 1, np.int64)
        np.cumsum(h.size, out=off[1:])
        self.off[l, : K + 1] = torch.as_tensor(off, dtype=torch.int32, device=dev)
        self.mem[l, : off[-1]] = torch.as_tensor(h.mem, dtype=torch.int32, device=dev)
        self.blocks[l] = [BlockRow(**vars(b)) for b in h.blocks]
        self.n_fine[l] = K
        self.max_size[l] = int(h.size.max()) if K else 0  # (the property flushes a pending refresh)
        if self.hierarchy:
            C = int(h.csize.size)
            if C > self.ccap:
                raise ValueError(f"ledger {l}: {C} coarse clusters > ccap {self.ccap}")
            self.ckc64[l, :C] = torch.as_tensor(h.ckc, dtype=torch.float64, device=dev)
            self.cvc64[l, :C] = torch.as_tensor(h.cvc, dtype=torch.float64, device=dev)
            self.ckc[l, :C] = self.ckc64[l, :C].to(self.dtype)
            self.cvc[l, :C] = self.cvc64[l, :C].to(self.dtype)
            self.csize[l, :C] = torch.as_tensor(h.csize, dtype=torch.int32, device=dev)
            self.ccount[l] = C
            self.coff[l, : C + 1] = torch.as_tensor(h.child_off, dtype=torch.int32, device=dev)
            self.child[l, : h.child.size] = torch.as_tensor(h.child, dtype=torch.int32, device=dev)
            self.n_coarse[l] = C

    def export(self, l: int, sink_end: int, buffer_start: int, total: int, splits: int) -> HostLedger:
        K = int(self.n_fine[l])
        off = self.off[l, : K + 1].cpu().numpy().astype(np.int64)
        h = HostLedger(sink_end, buffer_start, total, splits, [BlockRow(**vars(b)) for b in self.blocks[l]],
                       self.kc64[l, :K].cpu().numpy(), self.vc64[l, :K].cpu().numpy(),
                       self.size[l, :K].cpu().numpy().astype(np.int64),
                       self.mem[l, : off[-1]].cpu().numpy().astype(np.int64))
        if self.hierarchy:
            C = int(self.n_coarse[l])
            coff = self.coff[l, : C + 1].cpu().numpy().astype(np.int64)
            h.ckc = self.ckc64[l, :C].cpu().numpy()
            h.cvc = self.cvc64[l, :C].cpu().numpy()
            h.csize = self.csize[l, :C].cpu().numpy().astype(np.int64)
            h.child_off = coff
            h.child = self.child[l, : coff[-1]].cpu().numpy().astype(np.int64)
        return h
