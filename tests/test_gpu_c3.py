"""C3 serving path against the pinned oracle: the R1-Distill-Qwen-14B attention shape (40 q / 8 kv /
d128, G = 5) with the two-level hierarchy (r1 = 64, r2 = 8, p = 0.25) on a bf16 cache.

Four sealed blocks at reduced W, so every step's fused kernel mixes rejected coarse clusters and
rejected fine clusters in one rejected-centroid list (value-row codes < 0 and >= 0, gathered by
`tile::gather4` from the two levels) after the candidate-list logits (fine children of the promoted
coarse clusters, gathered rows) and the union-denominator selection (attention.py:293-351).  The online
updates run on the tcgen05 assignment (bf16, d = 128) and rebuild the final block's hierarchy.

Checked: ledgers bit-exact after prefill and after every update; per kv-head the selected token set,
selected / scored / rejected counts every step against the oracle given the centroids the GPU serves
(bf16-rounded copies of the same fp64 masters); outputs within 2e-3 relative L2 per q-head of the
oracle fed the stored bf16 K_rot / V, and within 1e-2 of it on the fp32 keys (queries at random-init
scale, |q| ~ sqrt(d)).
"""

import numpy as np
import pytest
import torch

from oracle import mpa_oracle as O
from paper_2506_13059_b200.core import EngineConfig, HeadLayout, HierarchyConfig, KvTrace, gen_synthetic
from tests.bridge import rel_err, rounded, to_oracle

pytestmark = pytest.mark.gpu


def _bf16(a):
    return torch.as_tensor(a).to(torch.bfloat16).float().numpy()


def _same_ledger(got, want, where):
    a, b = O.ledger_arrays(got), O.ledger_arrays(want)
    assert sorted(a) == sorted(b), where
    for k in a:
        assert np.array_equal(a[k], b[k]), (where, k)


def test_c3_hierarchical_bf16_d128_serving_path():
    from paper_2506_13059_b200 import pipeline as G

    lay = HeadLayout(40, 8, 128)
    raw = gen_synthetic(96, 4200, lay, 0.05, seed=17, decode_steps=100, query_gain=float(np.sqrt(128)))
    tr = KvTrace(lay, raw.prompt_len, _bf16(raw.keys), _bf16(raw.values), raw.queries)
    cfg = EngineConfig(block_size=1024, alpha=512, local_buffer=32, sink_tokens=10, token_budget=256,
                       hierarchy=HierarchyConfig(64, 8, 0.25), rope_theta=1e6, seed=17)
    st_g = G.prefill(tr, cfg, dtype=torch.bfloat16)
    st_o = O.prefill(tr, cfg, "multipole")
    eng = st_g.engine
    assert not eng.fused_lookup_path()  # the hierarchical staged kernels
    assert all(len(eng.led.blocks[h]) == 5 for h in range(8))  # 4 sealed + final
    for h in range(8):
        _same_ledger(to_oracle(eng.export_ledger(h)), st_o.ledgers[h], f"prefill h={h}")
    worst = worst_k = 0.0
    n_upd, mixed = 0, 0
    for t in range(100):
        pos = tr.prompt_len + t
        n = pos
        q = tr.queries[:, t]
        # the oracle on what the GPU serves: centroids rounded to bf16 (its lookup reads the bf16 copy),
        # and on what it stores: bf16 K_rot and V (kernel error only)
        ref_leds = [rounded(x, torch.bfloat16) for x in st_o.ledgers]
        keys = [tr.keys[h, :n] for h in range(8)]
        rk = [_bf16(O.rotate(tr.keys[h, :n], np.arange(n), 128, cfg.rope_theta)) for h in range(8)]
        want, rep_w = O.decode_step(q, ref_leds, keys, [tr.values[h, :n] for h in range(8)], n, t, cfg, lay)
        want_k, _ = O.decode_step(q, ref_leds, keys, [tr.values[h, :n] for h in range(8)], n, t, cfg, lay,
                                  rot_keys=rk)
        out_g, rep_g = G.step(st_g, q, tr.keys[:, pos], tr.values[:, pos])
        _, rep_o = O.step(st_o, q, tr.keys[:, pos], tr.values[:, pos])
        worst = max(worst, float(rel_err(out_g, want).max()))
        worst_k = max(worst_k, float(rel_err(out_g, want_k).max()))
        for h in range(8):
            assert np.array_equal(rep_g.selected_indices[h], rep_w.selected_indices[h]), (t, h)
            assert rep_g.per_head[h].selected_tokens == rep_w.per_head[h].selected_tokens
            assert rep_g.per_head[h].scored_centroids == rep_w.per_head[h].scored_centroids, (t, h)
            assert rep_g.per_head[h].rejected_centroids == rep_w.per_head[h].rejected_centroids, (t, h)
        # the rejected list mixes coarse (< 0) and fine (>= 0) value rows
        n_rej = eng.stats[1, :8].cpu().numpy()
        codes = eng.rej[:8].cpu().numpy()
        mixed += int(all((codes[h, :n_rej[h]] < 0).any() and (codes[h, :n_rej[h]] >= 0).any() for h in range(8)))
        assert rep_g.update_occurred == rep_o.update_occurred, t
        if rep_o.update_occurred:
            n_upd += 1
            for h in range(8):
                _same_ledger(to_oracle(eng.export_ledger(h)), st_o.ledgers[h], f"t={t} h={h}")
    assert n_upd >= 3
    assert mixed == 100
    assert worst_k <= 2e-3, worst_k  # the kernels' own arithmetic
    assert worst <= 1e-2, worst      # end to end incl. bf16 storage of K_rot / V
