"""Pin the CPU oracle to the reference: every fixture under tests/golden/ was produced by
running the real reference package (tests/golden/make_golden.py); the oracle restatement
must reproduce each array bit-for-bit."""

import hashlib
import os

import numpy as np
import pytest

from oracle import mpa_oracle as O
from paper_2506_13059_b200.core import EngineConfig, HeadLayout, HierarchyConfig, gen_synthetic

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, f"golden_{name}.npz")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def assert_ledger(g, prefix, led):
    mine = O.ledger_arrays(led)
    keys = sorted(k[len(prefix):] for k in g if k.startswith(prefix))
    assert keys, prefix
    for k in keys:
        assert k in mine, (prefix, k)
        assert np.array_equal(mine[k], g[prefix + k]), (prefix, k)


def test_rope_bitexact():
    g = load("rope")
    for th in (10000, 1000000):
        assert np.array_equal(O.rotate(g["rope_v"], g["rope_pos"], 16, float(th)), g[f"rope_out_{th}"])
    got = O.rotate(g["rope_v128"], np.array([0, 17, 32768, 65536, 131071]), 128, 1e6)
    assert np.array_equal(got, g["rope_out128"])


def test_gen_synthetic_bitexact():
    g = load("synthetic")
    tr = gen_synthetic(8, 600, HeadLayout(8, 2, 16), 0.05, seed=11, decode_steps=20)
    assert np.array_equal(tr.keys, g["syn_small_keys"])
    assert np.array_equal(tr.values, g["syn_small_values"])
    assert np.array_equal(tr.queries, g["syn_small_queries"])
    big = gen_synthetic(256, 8192, HeadLayout(32, 8, 128), 0.05, seed=0, decode_steps=32)
    assert [sha(big.keys), sha(big.values), sha(big.queries)] == list(g["syn_c1_sha"])


def test_kmeans_bitexact():
    g = load("kmeans")
    i = 0
    while f"km{i}_pts" in g:
        k, it, seed = (int(x) for x in g[f"km{i}_args"])
        lev = O.kmeans(g[f"km{i}_pts"], k, it, seed)
        assert np.array_equal(lev.kc, g[f"km{i}_kc"]), i
        assert np.array_equal(lev.sizes, g[f"km{i}_sizes"]), i
        assert np.array_equal(np.concatenate(lev.members), g[f"km{i}_members"]), i
        i += 1
    assert i == 7


def _ledger_cfg(hier=None):
    return EngineConfig(block_size=128, alpha=64, local_buffer=16, sink_tokens=8, token_budget=32,
                        tokens_per_centroid=8, hierarchy=hier, seed=5)


@pytest.mark.parametrize("tag,hier", [("flat", None), ("hier", HierarchyConfig(32, 8, 0.5))])
def test_prefill_and_updates_bitexact(tag, hier):
    g = load("ledgers")
    tr = gen_synthetic(6, 500, HeadLayout(2, 2, 8), 0.05, seed=5, decode_steps=200)
    cfg = _ledger_cfg(hier)
    for h in range(2):
        led = O.prefill_ledger(tr.keys[h, :500], tr.values[h, :500], 500, cfg, h)
        assert_ledger(g, f"led_{tag}_h{h}_prefill_", led)
    keys, values = tr.keys[0], tr.values[0]
    led = O.prefill_ledger(keys[:500], values[:500], 500, cfg, 0)
    n = 500
    for u in range(int(g[f"led_{tag}_nupd"])):
        n += 16
        led.total = n
        O.append_update(led, keys[:n], values[:n], cfg, np.random.default_rng(n), head=0)
        assert_ledger(g, f"led_{tag}_upd{u}_", led)
        O.audit(led, keys[:n], cfg, values=values[:n])
    assert led.splits >= 1


@pytest.mark.parametrize("tag,hier", [("flat", None), ("hp3", HierarchyConfig(32, 8, 0.3)),
                                      ("hp1", HierarchyConfig(32, 8, 1.0))])
def test_lookups_bitexact(tag, hier):
    g = load("lookups")
    tr = gen_synthetic(6, 400, HeadLayout(1, 1, 8), 0.05, seed=10, decode_steps=0)
    cfg = EngineConfig(block_size=128, alpha=64, local_buffer=16, sink_tokens=8, token_budget=48,
                       tokens_per_centroid=8, hierarchy=hier, seed=10)
    led = O.prefill_ledger(tr.keys[0], tr.values[0], 400, cfg, 0)
    assert_ledger(g, f"lk_{tag}_led_", led)
    for qi in range(6):
        p = f"lk_{tag}_q{qi}_"
        fn = O.flat_lookup if hier is None else O.hier_lookup
        lk = fn(g[p + "q"], led, cfg, 8)
        G = g[p + "q"].shape[0]
        assert np.array_equal(lk.sel_idx, g[p + "sel_idx"])
        assert np.array_equal(np.array(lk.sel_refs, np.int64).reshape(-1, 3), g[p + "sel_refs"])
        for nm, lst in (("frej", lk.fine_rej), ("crej", lk.coarse_rej)):
            assert np.array_equal(np.array([r[0] for r in lst], np.int64).reshape(-1, 3), g[p + nm + "_refs"])
            assert np.array_equal(np.array([r[3] for r in lst]).reshape(-1, G), g[p + nm + "_logits"])
        assert [lk.scored, lk.rejected] == list(g[p + "stats"])


def _check_run(g, prefix, reps):
    assert np.array_equal(np.stack([r.outputs for r in reps]), g[prefix + "outputs"])
    assert np.array_equal(np.array([r.update_occurred for r in reps]), g[prefix + "updates"])
    if prefix + "stats" in g:
        st = np.array([[[h.selected_tokens, h.scored_centroids, h.rejected_centroids] for h in r.per_head]
                       for r in reps])
        assert np.array_equal(st, g[prefix + "stats"])
        sel = [s for r in reps for s in r.selected_indices]
        assert np.array_equal(np.array([s.size for s in sel]), g[prefix + "sel_counts"])
        assert np.array_equal(np.concatenate(sel), g[prefix + "sel_concat"])


@pytest.mark.parametrize("mode", O.MODES)
def test_pipeline_runs_bitexact(mode):
    g = load("runs")
    small = gen_synthetic(8, 600, HeadLayout(8, 2, 16), 0.05, seed=11, decode_steps=20)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64, seed=11)
    _check_run(g, f"run_small_{mode}_", O.run(small, cfg, mode, max_steps=6 if mode == "oracle" else 20))


def test_full_budget_and_hier_runs_bitexact():
    g = load("runs")
    lay = HeadLayout(8, 2, 16)
    small = gen_synthetic(8, 600, lay, 0.05, seed=11, decode_steps=20)
    full = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=10**6, seed=11)
    _check_run(g, "run_small_fullbudget_", O.run(small, full, max_steps=6))
    tr = gen_synthetic(8, 600, lay, 0.05, seed=13, decode_steps=40)
    hcfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64,
                        hierarchy=HierarchyConfig(32, 8, 0.5), seed=13)
    _check_run(g, "run_hier_", O.run(tr, hcfg, max_steps=40))


def test_long_update_trajectory_bitexact():
    g = load("runs")
    lt = gen_synthetic(8, 1000, HeadLayout(4, 1, 16), 0.1, seed=3, decode_steps=400)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64, seed=3)
    st = O.prefill(lt, cfg)
    reps = []
    for t in range(lt.decode_steps):
        pos = lt.prompt_len + t
        out, rep = O.step(st, lt.queries[:, t], lt.keys[:, pos], lt.values[:, pos])
        rep.outputs = out
        reps.append(rep)
    _check_run(g, "run_long_", reps)
    assert_ledger(g, "run_long_final_led_", st.ledgers[0])
    assert st.ledgers[0].splits >= 1


def test_c1_shape_bitexact():
    g = load("c1")
    tr = gen_synthetic(256, 8192, HeadLayout(32, 8, 128), 0.05, seed=0, decode_steps=32)
    cfg = EngineConfig(tokens_per_centroid=32, token_budget=819, seed=0)
    st = O.prefill(tr, cfg)
    for h, led in enumerate(st.ledgers):
        lev = led.final.fine
        assert np.array_equal(lev.sizes.astype(np.int32), g[f"c1_h{h}_sizes"])
        assert np.array_equal(np.concatenate(lev.members).astype(np.int32), g[f"c1_h{h}_members"])
        assert sha(lev.kc) == str(g[f"c1_h{h}_kc_sha"])
        assert sha(lev.vc) == str(g[f"c1_h{h}_vc_sha"])
    reps = []
    for t in range(3):
        pos = tr.prompt_len + t
        out, rep = O.step(st, tr.queries[:, t], tr.keys[:, pos], tr.values[:, pos])
        rep.outputs = out
        reps.append(rep)
    _check_run(g, "c1_", reps)
