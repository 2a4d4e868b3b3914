"""On-device ledger audit (the invariants of clustering.py:548-623 `audit_ledger`), run with
torch ops on the engine's HBM state: partition of [0, total) by sinks + members + buffer,
contiguous W-sized sealed spans, final-block size window, centroid == member mean (key and
value, relative tolerance), and nearest-centroid assignment within each block (fp64)."""

from __future__ import annotations

import torch


class LedgerAuditError(AssertionError):
    pass


def audit_engine(eng, rel_tol: float = 1e-5, check_assignment: bool = True) -> None:
    cfg, led = eng.cfg, eng.led
    dev = eng.device
    for l in range(eng.L):
        s = l // eng.Hkv
        total, s0, bs = int(eng.cache_len[s]), int(eng.sink_end[s]), int(eng.buffer_start[s])
        rows = led.blocks[l]
        K = int(led.n_fine[l])
        off = led.off[l, : K + 1].long()
        nmem = int(off[-1]) if K else 0
        mem = led.mem[l, :nmem].long()
        if nmem != bs - s0:
            raise LedgerAuditError("token indices do not tile [0, total) exactly")
        seen = torch.zeros(total, dtype=torch.int32, device=dev)
        seen[:s0] += 1
        seen[bs:total] += 1
        seen.index_add_(0, mem, torch.ones_like(mem, dtype=torch.int32))
        if not bool((seen == 1).all()):
            raise LedgerAuditError("token indices do not tile [0, total) exactly")
        at = s0
        for r in rows[:-1]:
            if r.start != at or r.end - r.start != cfg.block_size:
                raise LedgerAuditError("sealed block spans are not contiguous W-sized")
            at = r.end
        F = rows[-1]
        if F.start != at or F.end != bs:
            raise LedgerAuditError("final block span inconsistent with buffer start")
        if F.end - F.start > cfg.block_size + cfg.alpha:
            raise LedgerAuditError("final block exceeds W + alpha")
        if eng.splits[l] > 0 and F.end - F.start < cfg.alpha:
            raise LedgerAuditError("final block shorter than alpha after a split")
        sizes = (off[1:] - off[:-1])
        if not bool((sizes == led.size[l, :K].long()).all()):
            raise LedgerAuditError("cluster size disagrees with member count")
        owner = torch.repeat_interleave(torch.arange(K, device=dev), sizes)
        keys = eng.k_raw[l, mem].double()
        vals = eng.values(l, mem).double()
        for cen, src, what in ((led.kc64[l, :K], keys, "key"), (led.vc64[l, :K], vals, "value")):
            acc = torch.zeros_like(cen).index_add_(0, owner, src)
            mean = acc / sizes[:, None].double()
            scale = max(1.0, float(cen.abs().max())) if K else 1.0
            if K and float((mean - cen).abs().max()) > rel_tol * scale:
                raise LedgerAuditError(f"{what} centroid drifted from member mean")
        if check_assignment:
            for r in rows:
                if r.fk == 0:
                    continue
                a, b = int(off[r.f0]), int(off[r.f0 + r.fk])
                pts = keys[a:b]
                c = led.kc64[l, r.f0:r.f0 + r.fk]
                dist = (pts * pts).sum(1)[:, None] + (c * c).sum(1)[None, :] - 2.0 * pts @ c.T
                near = dist.argmin(dim=1)
                if not bool((near == owner[a:b] - r.f0).all()):
                    raise LedgerAuditError("a member is not assigned to its nearest centroid")
