"""GPU parity of the decode path (K1, K9-K12 through the C ABI) against the pinned oracle.

Given the same ledger (built by the oracle, centroids rounded to what the GPU serves):
  * the selected token set equals the oracle's sel_idx bit-for-bit (ties: lowest cluster id),
  * per-head counts equal the oracle's (selected tokens, scored / rejected centroids),
  * outputs agree per q-head in relative L2: <= 1e-5 for fp32 caches, <= 1e-2 for bf16.
Mirrors reference tests: test_pipeline.py:84-98 (full budget == oracle), test_attention.py:126-138
(merge partition invariance), test_acceptance.py:94-132 (criterion 1).
"""

import numpy as np
import pytest
import torch

from oracle import mpa_oracle as O
from paper_2506_13059_b200.core import EngineConfig, HeadLayout, HierarchyConfig, gen_synthetic
from tests.bridge import rel_err, rounded, to_host

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.bfloat16: 1e-2}
# bf16 kernel error against the oracle fed the SAME stored cache (bf16 K_rot / V): the only
# remaining error is the kernel's own fp32 math, far below the storage effect.
KERNEL_TOL_BF16 = 2e-3
# bf16 K_rot storage vs the fp32 reference on gen_synthetic's deliberately peaked queries
# (query_gain = 12 sqrt(d)): SURVEY 7.3-5 measured up to 1.8e-2 from storage alone.
PEAKED_TOL_BF16 = 3e-2


def _stored(arr, dtype):
    return torch.as_tensor(arr, dtype=torch.float64).to(dtype).to(torch.float64).numpy()


def _engine(trace, cfg, dtype, ledgers, mode="multipole", n_seq=1):
    from paper_2506_13059_b200.engine import DecodeEngine

    lay = trace.layout
    P = trace.prompt_len
    eng = DecodeEngine(cfg, lay, n_seq, tcap=trace.total_len + 8, dtype=dtype, mode=mode)
    k = torch.as_tensor(trace.keys[:, :P]).cuda()[None].expand(n_seq, -1, -1, -1)
    v = torch.as_tensor(trace.values[:, :P]).cuda()[None].expand(n_seq, -1, -1, -1)
    eng.write_tokens(k, v)
    if ledgers is not None:
        eng.load_ledgers([to_host(led) for led in ledgers] * n_seq)
    else:
        eng.set_prompt_layout()
    return eng


def _replay(trace, cfg, dtype, steps, mode="multipole", check_sel=True, e2e_tol=None):
    lay, P = trace.layout, trace.prompt_len
    ledgers = [O.prefill_ledger(trace.keys[h, :P], trace.values[h, :P], P, cfg, h) for h in range(lay.num_kv_heads)]
    eng = _engine(trace, cfg, dtype, ledgers, mode)
    ref_ledgers = ledgers if dtype == torch.float32 else [rounded(x, dtype) for x in ledgers]
    if dtype == torch.float32:  # lookup reads fp64 masters; replacement reads fp32 value centroids
        ref_ledgers = [rounded(x, dtype, keys_too=False) for x in ledgers]
    keys = [trace.keys[h, :P].copy() for h in range(lay.num_kv_heads)]
    vals = [trace.values[h, :P].copy() for h in range(lay.num_kv_heads)]
    worst = worst_k = 0.0
    for t in range(steps):
        n = P + t
        q = trace.queries[:, t]
        out = eng.attend(torch.as_tensor(q).cuda()[None]).cpu().numpy()[0]
        want, rep = O.decode_step(q, ref_ledgers, keys, vals, n, t, cfg, lay, mode)
        worst = max(worst, float(rel_err(out, want).max()))
        if dtype != torch.float32:
            # the same step on exactly what the GPU stores (bf16 K_rot and V)
            rk = [_stored(O.rotate(keys[h], np.arange(n), lay.head_dim, cfg.rope_theta), dtype)
                  for h in range(lay.num_kv_heads)]
            sv = [_stored(vals[h], dtype) for h in range(lay.num_kv_heads)]
            want_k, _ = O.decode_step(q, ref_ledgers, keys, sv, n, t, cfg, lay, mode, rot_keys=rk)
            worst_k = max(worst_k, float(rel_err(out, want_k).max()))
        st = eng.head_stats()
        for h, led in enumerate(ref_ledgers):
            ns = min(led.sink_end, n)
            nb = n - led.buffer_start
            got_sel = np.sort(eng.tok[h, ns + nb: st[h, 0]].cpu().numpy())
            if check_sel:
                assert np.array_equal(got_sel, rep.selected_indices[h]), (t, h)
                assert st[h, 2] == rep.per_head[h].selected_tokens
                assert st[h, 1] == rep.per_head[h].rejected_centroids
        # append the step's token to both sides (no online update inside these short replays)
        kn = torch.as_tensor(trace.keys[:, n]).cuda()[None, :, None]
        vn = torch.as_tensor(trace.values[:, n]).cuda()[None, :, None]
        eng.write_tokens(kn, vn)
        for h in range(lay.num_kv_heads):
            keys[h] = np.concatenate([keys[h], trace.keys[h, n][None]])
            vals[h] = np.concatenate([vals[h], trace.values[h, n][None]])
            ref_ledgers[h].total += 1
    assert worst <= (e2e_tol or TOL[dtype]), worst
    if dtype != torch.float32:
        assert worst_k <= KERNEL_TOL_BF16, worst_k
    return worst


SMALL_CFG = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64, seed=11)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_small_trace_flat(dtype):
    tr = gen_synthetic(8, 600, HeadLayout(8, 2, 16), 0.05, seed=11, decode_steps=20)
    _replay(tr, SMALL_CFG, dtype, steps=12, e2e_tol=PEAKED_TOL_BF16 if dtype == torch.bfloat16 else None)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_small_trace_hierarchical(dtype):
    tr = gen_synthetic(8, 600, HeadLayout(8, 2, 16), 0.05, seed=13, decode_steps=40)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64,
                       hierarchy=HierarchyConfig(32, 8, 0.5), seed=13)
    _replay(tr, cfg, dtype, steps=12, e2e_tol=PEAKED_TOL_BF16 if dtype == torch.bfloat16 else None)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_flat_no_replacement(dtype):
    tr = gen_synthetic(8, 600, HeadLayout(8, 2, 16), 0.05, seed=11, decode_steps=20)
    _replay(tr, SMALL_CFG, dtype, steps=6, mode="flat-no-replacement",
            e2e_tol=PEAKED_TOL_BF16 if dtype == torch.bfloat16 else None)


@pytest.mark.parametrize("budget", [0, 1, 10**6])
def test_budget_edges(budget):
    # B = 0 selects nothing (test_attention.py:286-290); B >= total selects everything and the
    # result equals dense attention (test_pipeline.py:84-98).
    tr = gen_synthetic(8, 600, HeadLayout(8, 2, 16), 0.05, seed=11, decode_steps=20)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=budget, seed=11)
    _replay(tr, cfg, torch.float32, steps=3)


@pytest.mark.parametrize("layout", [HeadLayout(32, 8, 128), HeadLayout(40, 8, 128), HeadLayout(16, 4, 64)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_model_shapes(layout, dtype):
    # d=128/64 bf16 runs the tensor-core kernel (packed hi/lo for G=4, dual for G=5)
    tr = gen_synthetic(64, 3000, layout, 0.05, seed=3, decode_steps=8)
    cfg = EngineConfig(block_size=1024, local_buffer=32, token_budget=256, tokens_per_centroid=16, seed=3)
    _replay(tr, cfg, dtype, steps=4)


def test_c1_shape_fp32_and_bf16():
    # configs[0]: 32q/8kv/d128, 8K, r=32 (252 centroids), top-k 10% (B=819)
    tr = gen_synthetic(256, 8192, HeadLayout(32, 8, 128), 0.05, seed=0, decode_steps=32)
    cfg = EngineConfig(tokens_per_centroid=32, token_budget=819, seed=0)
    for dtype in (torch.float32, torch.bfloat16):
        _replay(tr, cfg, dtype, steps=3)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_split_invariance(dtype):
    tr = gen_synthetic(64, 3000, HeadLayout(32, 8, 128), 0.05, seed=5, decode_steps=4)
    cfg = EngineConfig(block_size=1024, local_buffer=32, token_budget=256, seed=5)
    P = tr.prompt_len
    ledgers = [O.prefill_ledger(tr.keys[h, :P], tr.values[h, :P], P, cfg, h) for h in range(8)]
    eng = _engine(tr, cfg, dtype, ledgers)
    q = torch.as_tensor(tr.queries[:, 0]).cuda()[None]
    outs = [eng.attend(q, n_split=s).clone().cpu().numpy() for s in (1, 2, 3, 7, 17, 64)]
    for o in outs[1:]:
        assert rel_err(o, outs[0]).max() < (1e-6 if dtype == torch.float32 else 1e-5)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("layout", [HeadLayout(8, 2, 16), HeadLayout(32, 8, 128)])
def test_dense_matches_oracle(dtype, layout):
    tr = gen_synthetic(16, 2500, layout, 0.1, seed=7, decode_steps=2)
    cfg = EngineConfig(block_size=1024, local_buffer=32, seed=7)
    eng = _engine(tr, cfg, dtype, None, mode="oracle")
    q = tr.queries[:, 0]
    out = eng.attend(torch.as_tensor(q).cuda()[None]).cpu().numpy()[0]
    P = tr.prompt_len
    pos = np.arange(P)
    want = np.stack([O.dense_attention(q[g], P, tr.keys[g // layout.group_size, :P],
                                       tr.values[g // layout.group_size, :P], pos, layout.head_dim, cfg.rope_theta)
                     for g in range(layout.num_q_heads)])
    assert rel_err(out, want).max() <= TOL[dtype]


def test_batched_sequences_identical():
    # n_seq > 1: every sequence replica must produce the same output as n_seq = 1
    tr = gen_synthetic(64, 3000, HeadLayout(32, 8, 128), 0.05, seed=5, decode_steps=4)
    cfg = EngineConfig(block_size=1024, local_buffer=32, token_budget=256, seed=5)
    P = tr.prompt_len
    ledgers = [O.prefill_ledger(tr.keys[h, :P], tr.values[h, :P], P, cfg, h) for h in range(8)]
    one = _engine(tr, cfg, torch.bfloat16, ledgers)
    four = _engine(tr, cfg, torch.bfloat16, ledgers, n_seq=4)
    q = torch.as_tensor(tr.queries[:, 0]).cuda()[None]
    a = one.attend(q).clone()
    b = four.attend(q.expand(4, -1, -1).contiguous())
    for s in range(4):
        assert rel_err(b[s].cpu().numpy(), a[0].cpu().numpy()).max() < 1e-5
