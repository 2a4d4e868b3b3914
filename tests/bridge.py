"""Test-only conversions between the oracle's ledgers (oracle/mpa_oracle.py) and the device
ledger's host view (paper_2506_13059_b200/ledger.py HostLedger)."""

from __future__ import annotations

import copy

import numpy as np
import torch

from oracle import mpa_oracle as O
from paper_2506_13059_b200.ledger import BlockRow, HostLedger


def to_host(led: O.LedgerO) -> HostLedger:
    d = led.blocks[0].fine.kc.shape[1]
    rows, kcs, vcs, sizes, mem = [], [], [], [], []
    ckc, cvc, csz, child, coff = [], [], [], [], [0]
    f0 = c0 = 0
    hier = all(b.coarse is not None for b in led.blocks)
    for b in led.blocks:
        fk = b.fine.k
        ck = b.coarse.k if hier else 0
        rows.append(BlockRow(b.start, b.end, f0, fk, c0, ck))
        kcs.append(b.fine.kc.reshape(-1, d))
        vcs.append(b.fine.vc.reshape(-1, d))
        sizes.extend(m.size for m in b.fine.members)
        mem.extend(b.fine.members)
        if hier:
            ckc.append(b.coarse.kc.reshape(-1, d))
            cvc.append(b.coarse.vc.reshape(-1, d))
            csz.extend(m.size for m in b.coarse.members)
            for ch in b.coarse.children:
                child.extend(f0 + int(c) for c in ch)
                coff.append(len(child))
        f0 += fk
        c0 += ck
    h = HostLedger(led.sink_end, led.buffer_start, led.total, led.splits, rows,
                   np.concatenate(kcs), np.concatenate(vcs), np.array(sizes, np.int64),
                   np.concatenate(mem) if mem else np.zeros(0, np.int64))
    if hier:
        h.ckc, h.cvc = np.concatenate(ckc), np.concatenate(cvc)
        h.csize = np.array(csz, np.int64)
        h.child_off = np.array(coff, np.int64)
        h.child = np.array(child, np.int64)
    return h


def to_oracle(h: HostLedger) -> O.LedgerO:
    blocks = []
    off = np.zeros(h.size.size + 1, np.int64)
    np.cumsum(h.size, out=off[1:])
    for r in h.blocks:
        ids = range(r.f0, r.f0 + r.fk)
        fine = O.Level(h.kc[r.f0:r.f0 + r.fk].copy(), h.vc[r.f0:r.f0 + r.fk].copy(),
                       [h.mem[off[i]:off[i + 1]].copy() for i in ids])
        coarse = None
        if h.csize is not None:
            kids = [[int(c) - r.f0 for c in h.child[h.child_off[j]:h.child_off[j + 1]]] for j in range(r.c0, r.c0 + r.ck)]
            cm = [np.sort(np.concatenate([fine.members[c] for c in k])) for k in kids]
            coarse = O.Level(h.ckc[r.c0:r.c0 + r.ck].copy(), h.cvc[r.c0:r.c0 + r.ck].copy(), cm, kids)
        blocks.append(O.BlockO(r.start, r.end, fine, coarse))
    return O.LedgerO(h.sink_end, blocks, h.buffer_start, h.total, h.splits)


def rounded(led: O.LedgerO, dtype: torch.dtype, keys_too: bool = True) -> O.LedgerO:
    """Copy of a ledger whose centroids are rounded through `dtype` (what the GPU serves)."""
    out = copy.deepcopy(led)

    def rnd(a):
        return torch.as_tensor(a, dtype=torch.float64).to(dtype).to(torch.float64).numpy()

    for b in out.blocks:
        for lev in (b.fine, b.coarse):
            if lev is None:
                continue
            if keys_too:
                lev.kc = rnd(lev.kc)
            lev.vc = rnd(lev.vc)
    return out


def rel_err(a, b) -> np.ndarray:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-300)
