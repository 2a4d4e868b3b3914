"""Paged serving cache (pipeline.py:26-52 `_KvStore` as a block-table pool): K_rot / V
live in page pools [n_pages, Hkv, page_size, d] with per-sequence block tables, pages handed out
from a free list (in shuffled order, as a long-running server would).  Every kernel that touches a
cached token row goes through the table: the fused decode step's append, the stream-K decode's
token gathers (TMA gather4 and the cp.async path), the fp32 FFMA decode, the dense decode and the
value means of the online update.  The paged engine must reproduce the flat engine bit-for-bit --
outputs at every step, selections, and the ledgers after online updates."""

import numpy as np
import pytest
import torch

from paper_2506_13059_b200.core import EngineConfig, HeadLayout, gen_synthetic
from tests.bridge import to_oracle

pytestmark = pytest.mark.gpu


def _engines(tr, cfg, dtype, variants):
    from paper_2506_13059_b200.engine import DecodeEngine

    P = tr.prompt_len
    out = []
    for kw in variants:
        e = DecodeEngine(cfg, tr.layout, 2, tcap=tr.total_len + 8, dtype=dtype, **kw)
        k = torch.as_tensor(tr.keys[:, :P]).cuda()[None].repeat(2, 1, 1, 1)
        v = torch.as_tensor(tr.values[:, :P]).cuda()[None].repeat(2, 1, 1, 1)
        e.write_tokens(k, v)
        e.prefill()
        out.append(e)
    return out


def _ledgers_equal(a, b):
    from oracle import mpa_oracle as O

    for h in range(a.L):
        x, y = O.ledger_arrays(to_oracle(a.export_ledger(h))), O.ledger_arrays(to_oracle(b.export_ledger(h)))
        assert sorted(x) == sorted(y), h
        for k in x:
            assert np.array_equal(x[k], y[k]), (h, k)


@pytest.mark.parametrize("dtype,d,group", [(torch.bfloat16, 128, 4), (torch.bfloat16, 64, 2), (torch.float32, 64, 4)])
def test_paged_matches_flat_across_updates(dtype, d, group):
    lay = HeadLayout(2 * group, 2, d)
    tr = gen_synthetic(8, 1000, lay, 0.1, seed=7, decode_steps=70)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64, seed=7)
    variants = [{}, {"page_size": 16, "page_order": "shuffled"},
                {"page_size": 64, "page_order": "shuffled", "use_graphs": False},
                {"page_size": 1, "page_order": "shuffled", "n_pages": 2 * 2 * (tr.total_len + 8)}]
    engs = _engines(tr, cfg, dtype, variants)
    assert engs[1].block_table is not None and engs[0].block_table is None
    # the pages really are scattered: consecutive logical pages are not consecutive physical ones
    bt = engs[1].block_table[0, :8].cpu().numpy()
    assert not np.array_equal(np.diff(bt), np.ones(7))
    P = tr.prompt_len
    n_upd = 0
    for t in range(70):
        q = torch.as_tensor(tr.queries[:, t]).cuda()[None].repeat(2, 1, 1)
        kn = torch.as_tensor(tr.keys[:, P + t]).cuda()[None].repeat(2, 1, 1)
        vn = torch.as_tensor(tr.values[:, P + t]).cuda()[None].repeat(2, 1, 1)
        outs = [e.step(q, kn, vn).clone() for e in engs]
        for i in range(1, len(engs)):
            assert torch.equal(outs[0], outs[i]), (t, i)
        n_upd += engs[0].last_update is not None
    assert n_upd >= 3
    for e in engs[1:]:
        _ledgers_equal(engs[0], e)
        assert torch.equal(engs[0].stats, e.stats)
    # the rows behind the table hold exactly the flat cache's rows
    n = int(engs[0].cache_len[0])
    for l in range(engs[0].L):
        t = torch.arange(n)
        assert torch.equal(engs[0].values(l, t), engs[1].values(l, t))
        assert torch.equal(engs[0].keys_rotated(l, t), engs[3].keys_rotated(l, t))
    # dense decode through the table
    q = torch.as_tensor(tr.queries[:, 0]).cuda()[None].repeat(2, 1, 1)
    assert torch.equal(engs[0].attend_dense(q).clone(), engs[1].attend_dense(q).clone())


def test_c2_shape_paged_step_matches_flat():
    # the serving shape of the benchmark (32q/8kv/d128, bf16, fused decode step), 4K context,
    # 16-token pages in shuffled order: step outputs bit-identical to the flat cache
    lay = HeadLayout(32, 8, 128)
    tr = gen_synthetic(16, 4096, lay, 0.1, seed=3, decode_steps=24)
    cfg = EngineConfig(block_size=1024, alpha=512, local_buffer=64, sink_tokens=10, token_budget=256,
                       tokens_per_centroid=16, rope_theta=1e6, seed=3)
    flat, paged = _engines(tr, cfg, torch.bfloat16, [{}, {"page_size": 16, "page_order": "shuffled"}])
    assert flat.fused_lookup_path() and paged.fused_lookup_path()
    P = tr.prompt_len
    for t in range(24):
        q = torch.as_tensor(tr.queries[:, t]).cuda()[None].repeat(2, 1, 1)
        kn = torch.as_tensor(tr.keys[:, P + t]).cuda()[None].repeat(2, 1, 1)
        vn = torch.as_tensor(tr.values[:, P + t]).cuda()[None].repeat(2, 1, 1)
        assert torch.equal(flat.step(q, kn, vn).clone(), paged.step(q, kn, vn).clone()), t


def test_page_pool_exhaustion_is_an_error():
    from paper_2506_13059_b200.engine import DecodeEngine

    lay = HeadLayout(4, 2, 64)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64)
    e = DecodeEngine(cfg, lay, 2, tcap=512, dtype=torch.bfloat16, page_size=64, n_pages=5)
    k = torch.zeros(2, 2, 128, 64, device="cuda")
    e.write_tokens(k, k)  # 2 pages per sequence
    with pytest.raises(RuntimeError, match="exhausted"):
        e.write_tokens(k, k)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_paged_hierarchical_matches_flat(dtype):
    # 2-level hierarchy (coarse rejected rows in the work lists, staged lookup) on a paged cache
    from paper_2506_13059_b200.core import HierarchyConfig

    lay = HeadLayout(10, 2, 128)
    tr = gen_synthetic(8, 1400, lay, 0.1, seed=17, decode_steps=40)
    cfg = EngineConfig(block_size=512, alpha=256, local_buffer=16, sink_tokens=5, token_budget=96,
                       tokens_per_centroid=8, seed=17, hierarchy=HierarchyConfig(32, 4, 0.5))
    flat, paged = _engines(tr, cfg, dtype, [{}, {"page_size": 32, "page_order": "shuffled"}])
    P = tr.prompt_len
    n_upd = 0
    for t in range(40):
        q = torch.as_tensor(tr.queries[:, t]).cuda()[None].repeat(2, 1, 1)
        kn = torch.as_tensor(tr.keys[:, P + t]).cuda()[None].repeat(2, 1, 1)
        vn = torch.as_tensor(tr.values[:, P + t]).cuda()[None].repeat(2, 1, 1)
        assert torch.equal(flat.step(q, kn, vn).clone(), paged.step(q, kn, vn).clone()), t
        n_upd += flat.last_update is not None
    assert n_upd >= 2
    _ledgers_equal(flat, paged)
