"""Selection and output parity of the single-launch serving decode step at BENCHMARK scale (C2: Qwen3-8B
shape, 32K context, r=16, ~2040 centroids per kv-head) against the pinned oracle, through every cluster
size of the step kernel (mpa_decode_step: C = 16, 8, 4, 1 CTAs per ledger at batch 1, 2, 4, 16).

The ledgers are synthetic but well-formed (contiguous W-blocks partitioned into clusters whose key /
value centroids are the exact member means, C2's cluster-size statistics); the oracle is handed the
same ledgers with centroids rounded to what the GPU serves (bf16).  Checked per kv-head: the selected
token set (ties: lowest cluster id), selected / rejected counts, and outputs against the oracle fed the
stored bf16 cache (reference: attention.py:192-207, 267-290, 354-375, 410-552).
"""

import numpy as np
import pytest
import torch

from oracle import mpa_oracle as O
from paper_2506_13059_b200.core import EngineConfig, HeadLayout
from tests.bridge import rel_err, rounded, to_host

pytestmark = pytest.mark.gpu

LAY = HeadLayout(32, 8, 128)
CTX = 32768


def _ledger(rng, ctx, cfg, dup_frac=0.0):
    """Blocks of W tokens after the sinks, each partitioned at random into ceil(len / r) clusters."""
    d = LAY.head_dim
    keys = rng.standard_normal((ctx, d)).astype(np.float32)
    vals = rng.standard_normal((ctx, d)).astype(np.float32)
    s0 = cfg.sink_tokens
    b0 = ctx - cfg.local_buffer
    blocks, start = [], s0
    while start < b0:
        end = min(start + cfg.block_size, b0)
        n = end - start
        k = -(-n // cfg.fine_ratio)
        lab = np.concatenate([np.arange(k), rng.integers(0, k, n - k)])
        rng.shuffle(lab)
        mem = [np.flatnonzero(lab == c).astype(np.int64) + start for c in range(k)]
        kc = np.stack([keys[m].astype(np.float64).mean(0) for m in mem])
        vc = np.stack([vals[m].astype(np.float64).mean(0) for m in mem])
        if dup_frac:
            # duplicated centroids AND sizes: exact score ties that only the id tie-break orders
            src = rng.choice(k, int(dup_frac * k), replace=False)
            for a, b in zip(src[::2], src[1::2]):
                kc[b] = kc[a]
                keep = min(mem[a].size, mem[b].size)
                mem[a], mem[b] = mem[a][:keep], mem[b][:keep]
            # tokens dropped from a trimmed cluster join a fresh singleton cluster
            used = np.zeros(ctx, bool)
            for m in mem:
                used[m] = True
            spare = np.flatnonzero(~used[start:end]) + start
            for t in spare:
                mem.append(np.array([t], np.int64))
            kc = np.concatenate([kc, keys[spare].astype(np.float64)]) if spare.size else kc
            vc = np.concatenate([vc, vals[spare].astype(np.float64)]) if spare.size else vc
        blocks.append(O.BlockO(start, end, O.Level(kc, vc, mem)))
        start = end
    led = O.LedgerO(s0, blocks, b0, ctx)
    return keys, vals, led


def _run(n_seq, budget, dup_frac=0.0, seed=0):
    from paper_2506_13059_b200.engine import DecodeEngine

    cfg = EngineConfig(block_size=8192, alpha=4096, local_buffer=128, sink_tokens=10, tokens_per_centroid=16,
                       token_budget=budget, rope_theta=1e6, seed=seed)
    rng = np.random.default_rng(seed)
    heads = [_ledger(rng, CTX, cfg, dup_frac) for _ in range(LAY.num_kv_heads)]
    keys = np.stack([h[0] for h in heads])
    vals = np.stack([h[1] for h in heads])
    ledgers = [h[2] for h in heads]
    eng = DecodeEngine(cfg, LAY, n_seq, tcap=CTX + 8, dtype=torch.bfloat16,
                       kcap=max(O._flat(x, False)[2].size for x in ledgers) + 64)
    assert eng.fused_lookup_path()
    k = torch.as_tensor(keys).cuda()[None].expand(n_seq, -1, -1, -1)
    v = torch.as_tensor(vals).cuda()[None].expand(n_seq, -1, -1, -1)
    eng.write_tokens(k, v)
    eng.load_ledgers([to_host(x) for x in ledgers] * n_seq)
    q = rng.standard_normal((LAY.num_q_heads, LAY.head_dim)).astype(np.float32)
    out = eng.attend(torch.as_tensor(q).cuda()[None].expand(n_seq, -1, -1).contiguous()).cpu().numpy()
    ref = [rounded(x, torch.bfloat16) for x in ledgers]
    st = eng.head_stats()
    tok = eng.tok.cpu().numpy()
    # the oracle on exactly what the GPU stores (bf16 K_rot / V)
    rk = [torch.as_tensor(O.rotate(keys[h], np.arange(CTX), LAY.head_dim, cfg.rope_theta)).to(torch.bfloat16)
          .double().numpy() for h in range(LAY.num_kv_heads)]
    sv = [torch.as_tensor(vals[h]).to(torch.bfloat16).double().numpy() for h in range(LAY.num_kv_heads)]
    want, rep = O.decode_step(q, ref, [keys[h] for h in range(8)], sv, CTX, 0, cfg, LAY, rot_keys=rk)
    for s in range(n_seq):
        for h in range(LAY.num_kv_heads):
            l = s * LAY.num_kv_heads + h
            ns, nb = cfg.sink_tokens, CTX - ref[h].buffer_start
            got = np.sort(tok[l, ns + nb: st[l, 0]])
            assert np.array_equal(got, rep.selected_indices[h]), (n_seq, s, h)
            assert st[l, 2] == rep.per_head[h].selected_tokens
            assert st[l, 1] == rep.per_head[h].rejected_centroids
            assert st[l, 3] == len(rep.per_head[h].selected_refs)
        assert rel_err(out[s], want).max() < 2e-3, (n_seq, s)
    return rep


@pytest.mark.parametrize("n_seq", [1, 2, 4, 16])
def test_c2_selection_every_cluster_size(n_seq):
    _run(n_seq, 512)


@pytest.mark.parametrize("budget", [128, 3277])
def test_c2_selection_budgets(budget):
    _run(1, budget)


def test_c2_selection_exact_ties():
    # a third of the clusters come in pairs with identical centroids and sizes
    rep = _run(4, 512, dup_frac=0.34, seed=3)
    assert all(h.selected_tokens >= 512 for h in rep.per_head)


@pytest.mark.parametrize("budget", [0, 1, 10**9])
def test_c2_selection_budget_edges(budget):
    rep = _run(2, budget, seed=5)
    if budget == 0:
        assert all(h.selected_tokens == 0 for h in rep.per_head)
    if budget == 10**9:
        assert all(h.rejected_centroids == 0 for h in rep.per_head)


def test_c2_staged_lookup_matches_single_launch():
    # the staged kernels (logits -> selection -> lists, taken when the single-launch step does not
    # fit the device, e.g. C5's 8K centroids per ledger at batch 16) produce the same lists and outputs
    from paper_2506_13059_b200.engine import DecodeEngine

    cfg = EngineConfig(block_size=8192, alpha=4096, local_buffer=128, sink_tokens=10, tokens_per_centroid=16,
                       token_budget=512, rope_theta=1e6, seed=11)
    rng = np.random.default_rng(11)
    heads = [_ledger(rng, CTX, cfg) for _ in range(LAY.num_kv_heads)]
    eng = DecodeEngine(cfg, LAY, 2, tcap=CTX + 8, dtype=torch.bfloat16,
                       kcap=max(O._flat(x[2], False)[2].size for x in heads) + 64)
    k = torch.as_tensor(np.stack([h[0] for h in heads])).cuda()[None].expand(2, -1, -1, -1)
    v = torch.as_tensor(np.stack([h[1] for h in heads])).cuda()[None].expand(2, -1, -1, -1)
    eng.write_tokens(k, v)
    eng.load_ledgers([to_host(h[2]) for h in heads] * 2)
    q = torch.as_tensor(rng.standard_normal((2, LAY.num_q_heads, LAY.head_dim)).astype(np.float32)).cuda()
    assert eng.fused_lookup_path()
    out1 = eng.attend(q).clone()
    st1, tok1, w1 = eng.stats.clone(), eng.tok.clone(), eng.rej_w.clone()
    eng.rotate(q, exact=True, lookup=False)
    eng.lookup(q, staged=True)
    out2 = eng.fused().clone()
    assert torch.equal(st1, eng.stats)
    for l in range(eng.L):
        n = int(st1[0, l])
        assert torch.equal(tok1[l, :n].sort().values, eng.tok[l, :n].sort().values), l
    kc = int(eng.led.count.max())
    a, b = w1[:, :kc].cpu().numpy(), eng.rej_w[:, :kc].cpu().numpy()
    assert np.array_equal(np.isinf(a), np.isinf(b))  # the same selected rows
    fin = np.isfinite(a)
    assert np.allclose(a[fin], b[fin], rtol=1e-6, atol=1e-6)
    assert rel_err(out1.cpu().numpy(), out2.cpu().numpy()).max() < 1e-5


def test_oversized_step_falls_back_to_staged_kernels():
    # 128 ledgers of ~2.5K centroids: the single-launch step's one-wave cluster grid does not fit
    # (mpa_decode_step_fits), so the engine takes the staged kernels -- selections still exact
    from paper_2506_13059_b200.engine import DecodeEngine

    ctx = 5200
    cfg = EngineConfig(block_size=2048, alpha=1024, local_buffer=64, sink_tokens=10, tokens_per_centroid=2,
                       token_budget=256, rope_theta=1e6, seed=13)
    rng = np.random.default_rng(13)
    heads = [_ledger(rng, ctx, cfg) for _ in range(LAY.num_kv_heads)]
    n_seq = 16
    kcap = max(O._flat(x[2], False)[2].size for x in heads) + 64
    eng = DecodeEngine(cfg, LAY, n_seq, tcap=ctx + 8, dtype=torch.bfloat16, kcap=kcap)
    k = torch.as_tensor(np.stack([h[0] for h in heads])).cuda()[None].expand(n_seq, -1, -1, -1)
    v = torch.as_tensor(np.stack([h[1] for h in heads])).cuda()[None].expand(n_seq, -1, -1, -1)
    eng.write_tokens(k, v)
    eng.load_ledgers([to_host(h[2]) for h in heads] * n_seq)
    assert int(eng.led.n_fine.max()) > 2300
    assert not eng.fused_lookup_path()
    q = rng.standard_normal((LAY.num_q_heads, LAY.head_dim)).astype(np.float32)
    out = eng.attend(torch.as_tensor(q).cuda()[None].expand(n_seq, -1, -1).contiguous()).cpu().numpy()
    ref = [rounded(h[2], torch.bfloat16) for h in heads]
    rk = [torch.as_tensor(O.rotate(heads[h][0], np.arange(ctx), LAY.head_dim, cfg.rope_theta)).to(torch.bfloat16)
          .double().numpy() for h in range(LAY.num_kv_heads)]
    sv = [torch.as_tensor(heads[h][1]).to(torch.bfloat16).double().numpy() for h in range(LAY.num_kv_heads)]
    want, rep = O.decode_step(q, ref, [h[0] for h in heads], sv, ctx, 0, cfg, LAY, rot_keys=rk)
    st, tok = eng.head_stats(), eng.tok.cpu().numpy()
    for s in (0, n_seq - 1):
        for h in range(LAY.num_kv_heads):
            l = s * LAY.num_kv_heads + h
            ns, nb = cfg.sink_tokens, ctx - ref[h].buffer_start
            assert np.array_equal(np.sort(tok[l, ns + nb: st[l, 0]]), rep.selected_indices[h]), (s, h)
        assert rel_err(out[s], want).max() < 2e-3
