"""GPU clustering (K2-K8) and the end-to-end pipeline against the pinned oracle.

* prefill ledgers (blockwise k-means, hierarchy) equal the oracle's bit-for-bit: spans,
  cluster order, sizes, members, fp64 key/value centroids, coarse children;
* online updates (sequential assignment + Lloyd refinement + split/settle + hierarchy rebuild)
  over long replays equal the oracle's ledgers after every update;
* `pipeline.run` reproduces the oracle's outputs (fp32: 1e-5) and selections on the reference's
  own test scenarios (test_pipeline.py, test_clustering.py:179-194, acceptance criterion 6).
"""

import numpy as np
import pytest
import torch

from oracle import mpa_oracle as O
from paper_2506_13059_b200.core import EngineConfig, HeadLayout, HierarchyConfig, KvTrace, gen_synthetic
from tests.bridge import rel_err, to_oracle

pytestmark = pytest.mark.gpu


def _bf16(a):
    return torch.as_tensor(a).to(torch.bfloat16).float().numpy()


def _engine_prefill(trace, cfg, dtype, mode="multipole"):
    from paper_2506_13059_b200.engine import DecodeEngine

    P = trace.prompt_len
    eng = DecodeEngine(cfg, trace.layout, 1, tcap=trace.total_len + 8, dtype=dtype, mode=mode)
    eng.write_tokens(torch.as_tensor(trace.keys[:, :P]).cuda()[None], torch.as_tensor(trace.values[:, :P]).cuda()[None])
    eng.prefill()
    return eng


def _assert_same_ledger(got: O.LedgerO, want: O.LedgerO, where=""):
    a, b = O.ledger_arrays(got), O.ledger_arrays(want)
    assert sorted(a) == sorted(b), where
    for k in a:
        assert np.array_equal(a[k], b[k]), (where, k)


def _as_dtype_trace(trace, dtype):
    if dtype == torch.float32:
        return trace
    return KvTrace(trace.layout, trace.prompt_len, _bf16(trace.keys), _bf16(trace.values), trace.queries)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("hier", [None, HierarchyConfig(32, 8, 0.5)])
def test_prefill_ledgers_bitexact(dtype, hier):
    tr = _as_dtype_trace(gen_synthetic(6, 500, HeadLayout(2, 2, 8), 0.05, seed=5, decode_steps=200), dtype)
    cfg = EngineConfig(block_size=128, alpha=64, local_buffer=16, sink_tokens=8, token_budget=32,
                       tokens_per_centroid=8, hierarchy=hier, seed=5)
    eng = _engine_prefill(tr, cfg, dtype)
    for h in range(2):
        want = O.prefill_ledger(tr.keys[h, :500], tr.values[h, :500], 500, cfg, h)
        _assert_same_ledger(to_oracle(eng.export_ledger(h)), want, f"head {h}")


def test_kmeans_degenerate_duplicates_and_empty_repair():
    # duplicate-heavy points exercise _repair_empty and the sizes[big] <= 1 stop (test_clustering.py:69-72)
    lay = HeadLayout(1, 1, 4)
    keys = np.zeros((1, 60, 4), np.float32)
    keys[0, 30:] = 1.0
    vals = np.random.default_rng(0).standard_normal((1, 60, 4)).astype(np.float32)
    tr = KvTrace(lay, 60, keys, vals, np.zeros((1, 0, 4), np.float32))
    cfg = EngineConfig(block_size=64, local_buffer=2, sink_tokens=2, tokens_per_centroid=4, seed=1)
    eng = _engine_prefill(tr, cfg, torch.float32)
    want = O.prefill_ledger(keys[0], vals[0], 60, cfg, 0)
    _assert_same_ledger(to_oracle(eng.export_ledger(0)), want)


def test_c1_prefill_bitexact():
    tr = gen_synthetic(256, 8192, HeadLayout(32, 8, 128), 0.05, seed=0, decode_steps=32)
    cfg = EngineConfig(tokens_per_centroid=32, token_budget=819, seed=0)
    eng = _engine_prefill(tr, cfg, torch.float32)
    for h in range(8):
        want = O.prefill_ledger(tr.keys[h, :8192], tr.values[h, :8192], 8192, cfg, h)
        _assert_same_ledger(to_oracle(eng.export_ledger(h)), want, f"head {h}")


def _run_both(tr, cfg, steps, dtype=torch.float32, mode="multipole", check_ledgers_every_update=True):
    from paper_2506_13059_b200 import pipeline as G

    st_g = G.prefill(tr, cfg, mode=mode, dtype=dtype)
    st_o = O.prefill(tr, cfg, mode)
    worst = 0.0
    n_upd = 0
    for t in range(steps):
        pos = tr.prompt_len + t
        args = (tr.queries[:, t], tr.keys[:, pos], tr.values[:, pos])
        out_g, rep_g = G.step(st_g, *args)
        out_o, rep_o = O.step(st_o, *args)
        worst = max(worst, float(rel_err(out_g, out_o).max()))
        assert rep_g.update_occurred == rep_o.update_occurred, t
        if mode != "oracle":
            for h in range(tr.layout.num_kv_heads):
                assert np.array_equal(rep_g.selected_indices[h], rep_o.selected_indices[h]), (t, h)
                assert rep_g.per_head[h].selected_tokens == rep_o.per_head[h].selected_tokens
                assert rep_g.per_head[h].scored_centroids == rep_o.per_head[h].scored_centroids, (t, h)
                assert rep_g.per_head[h].rejected_centroids == rep_o.per_head[h].rejected_centroids
        if rep_o.update_occurred:
            n_upd += 1
            if check_ledgers_every_update:
                for h in range(tr.layout.num_kv_heads):
                    _assert_same_ledger(to_oracle(st_g.engine.export_ledger(h)), st_o.ledgers[h], f"t={t} h={h}")
    return worst, n_upd, st_g, st_o


@pytest.mark.parametrize("mode", ["multipole", "flat-no-replacement", "positional-baseline", "oracle"])
def test_pipeline_small_trace(mode):
    tr = gen_synthetic(8, 600, HeadLayout(8, 2, 16), 0.05, seed=11, decode_steps=20)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64, seed=11)
    worst, n_upd, _, _ = _run_both(tr, cfg, 20, mode=mode)
    assert worst < 1e-5, worst
    if mode != "oracle":
        assert n_upd == 1


def test_pipeline_long_trajectory_with_splits():
    # online updates every L steps with two sliding-window splits (C4 analogue at desk scale)
    tr = gen_synthetic(8, 1000, HeadLayout(4, 1, 16), 0.1, seed=3, decode_steps=400)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64, seed=3)
    worst, n_upd, st_g, _ = _run_both(tr, cfg, 400)
    assert worst < 1e-5, worst
    assert n_upd == 25
    assert st_g.engine.splits[0] >= 1


def test_pipeline_hierarchical_updates():
    tr = gen_synthetic(8, 600, HeadLayout(8, 2, 16), 0.05, seed=13, decode_steps=40)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64,
                       hierarchy=HierarchyConfig(32, 8, 0.5), seed=13)
    worst, n_upd, _, _ = _run_both(tr, cfg, 40)
    assert worst < 1e-5, worst
    assert n_upd >= 2


def test_pipeline_hierarchical_splits():
    tr = gen_synthetic(8, 700, HeadLayout(4, 1, 16), 0.1, seed=21, decode_steps=300)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64,
                       hierarchy=HierarchyConfig(32, 8, 0.25), seed=21)
    worst, n_upd, st_g, _ = _run_both(tr, cfg, 300)
    assert worst < 1e-5, worst
    assert st_g.engine.splits[0] >= 1


def test_audit_after_updates():
    from paper_2506_13059_b200 import pipeline as G

    tr = gen_synthetic(8, 1000, HeadLayout(4, 1, 16), 0.1, seed=3, decode_steps=200)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64, seed=3)
    reps = G.run(tr, cfg, audit=True, max_steps=200)
    assert sum(r.update_occurred for r in reps) == 12


def test_update_cadence_and_attend_before_append():
    # test_pipeline.py:44-53 and :71-81
    from paper_2506_13059_b200 import pipeline as G

    tr = gen_synthetic(8, 600, HeadLayout(8, 2, 16), 0.05, seed=11, decode_steps=20)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64, seed=11)
    reps = G.run(tr, cfg, max_steps=20)
    ups = [r.step for r in reps if r.update_occurred]
    assert ups and ups[0] == cfg.local_buffer - 1
    a = G.prefill(tr, cfg)
    b = G.prefill(tr, cfg)
    q, pos = tr.queries[:, 0], tr.prompt_len
    oa, _ = G.step(a, q, tr.keys[:, pos], tr.values[:, pos])
    ob, _ = G.step(b, q, -tr.keys[:, pos], -tr.values[:, pos])
    assert np.array_equal(oa, ob)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_engine_step_graph_matches_eager(dtype):
    """DecodeEngine.step replayed as a CUDA graph (attend + device-side append) gives the same
    outputs, selections and ledgers as the eager launch sequence, across online updates."""
    from paper_2506_13059_b200.engine import DecodeEngine

    tr = gen_synthetic(8, 1000, HeadLayout(8, 2, 64), 0.1, seed=5, decode_steps=60)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64, seed=5)
    P = tr.prompt_len
    engs = []
    for graphs in (True, False):
        e = DecodeEngine(cfg, tr.layout, 2, tcap=tr.total_len + 8, dtype=dtype, use_graphs=graphs)
        k = torch.as_tensor(tr.keys[:, :P]).cuda()[None].repeat(2, 1, 1, 1)
        v = torch.as_tensor(tr.values[:, :P]).cuda()[None].repeat(2, 1, 1, 1)
        e.write_tokens(k, v)
        e.prefill()
        engs.append(e)
    n_upd = 0
    for t in range(60):
        q = torch.as_tensor(tr.queries[:, t]).cuda()[None].repeat(2, 1, 1)
        kn = torch.as_tensor(tr.keys[:, P + t]).cuda()[None].repeat(2, 1, 1)
        vn = torch.as_tensor(tr.values[:, P + t]).cuda()[None].repeat(2, 1, 1)
        outs = [e.step(q, kn, vn).clone() for e in engs]
        assert torch.equal(outs[0], outs[1]), t
        assert np.array_equal(engs[0].cache_len, engs[1].cache_len)
        assert torch.equal(engs[0].cache_len_d, engs[1].cache_len_d)
        n_upd += engs[0].last_update is not None
    assert n_upd >= 3
    for h in range(engs[0].L):
        _assert_same_ledger(to_oracle(engs[0].export_ledger(h)), to_oracle(engs[1].export_ledger(h)), f"h={h}")


def test_bf16_d128_tensor_core_clustering_bitexact(monkeypatch):
    # bf16 keys with d = 128 take the tcgen05 assignment (persistent paired kernel + fp64 recheck):
    # prefill and every online update must give the oracle's ledgers bit-for-bit on the same keys
    from paper_2506_13059_b200 import clustering as GC
    from paper_2506_13059_b200 import pipeline as G

    used = []
    orig = GC.KMeansBatch.lloyd

    def lloyd(self):
        used.append(self.tc_ws is not None)
        return orig(self)

    monkeypatch.setattr(GC.KMeansBatch, "lloyd", lloyd)
    tr = _as_dtype_trace(gen_synthetic(16, 2048, HeadLayout(8, 2, 128), 0.05, seed=9, decode_steps=40),
                         torch.bfloat16)
    cfg = EngineConfig(block_size=1024, alpha=512, local_buffer=16, sink_tokens=5, token_budget=128,
                       tokens_per_centroid=8, seed=9)
    st_g = G.prefill(tr, cfg, dtype=torch.bfloat16)
    st_o = O.prefill(tr, cfg, "multipole")
    for h in range(2):
        _assert_same_ledger(to_oracle(st_g.engine.export_ledger(h)), st_o.ledgers[h], f"prefill h={h}")
    n_upd = 0
    for t in range(40):
        pos = tr.prompt_len + t
        args = (tr.queries[:, t], tr.keys[:, pos], tr.values[:, pos])
        _, rep_g = G.step(st_g, *args)
        _, rep_o = O.step(st_o, *args)
        assert rep_g.update_occurred == rep_o.update_occurred, t
        if rep_o.update_occurred:
            n_upd += 1
            for h in range(2):
                _assert_same_ledger(to_oracle(st_g.engine.export_ledger(h)), st_o.ledgers[h], f"t={t} h={h}")
    assert n_upd >= 2
    assert used and all(used), used  # every Lloyd call ran on the tensor cores


@pytest.mark.parametrize("use_graphs", [True, False])
def test_step_host_matches_step(use_graphs):
    """DecodeEngine.step_host (pinned host buffers; with a captured step graph one native call:
    copies in, the graph, the copy out) gives the device-buffer step's outputs bit-for-bit, and the
    same ledgers, across online updates."""
    from paper_2506_13059_b200.engine import DecodeEngine

    tr = gen_synthetic(8, 1000, HeadLayout(8, 2, 128), 0.1, seed=6, decode_steps=60)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64,
                       tokens_per_centroid=8, seed=6)
    P = tr.prompt_len
    engs = []
    for _ in range(2):
        e = DecodeEngine(cfg, tr.layout, 2, tcap=tr.total_len + 8, dtype=torch.bfloat16, use_graphs=use_graphs)
        k = torch.as_tensor(tr.keys[:, :P]).cuda()[None].repeat(2, 1, 1, 1)
        v = torch.as_tensor(tr.values[:, :P]).cuda()[None].repeat(2, 1, 1, 1)
        e.write_tokens(k, v)
        e.prefill()
        engs.append(e)
    oh = torch.empty(2, 8, 128, dtype=torch.float32).pin_memory()
    n_upd = 0
    for t in range(60):
        q = torch.as_tensor(tr.queries[:, t]).float()[None].repeat(2, 1, 1).contiguous()
        kn = torch.as_tensor(tr.keys[:, P + t]).float()[None].repeat(2, 1, 1).contiguous()
        vn = torch.as_tensor(tr.values[:, P + t]).float()[None].repeat(2, 1, 1).contiguous()
        ref = engs[0].step(q.cuda(), kn.cuda(), vn.cuda()).cpu()
        engs[1].step_host(q.pin_memory(), kn.pin_memory(), vn.pin_memory(), oh)
        torch.cuda.synchronize()
        assert torch.equal(ref, oh), t
        n_upd += engs[0].last_update is not None
    assert n_upd >= 3
    assert engs[1].n_captures >= 1 or not use_graphs
    for h in range(engs[0].L):
        _assert_same_ledger(to_oracle(engs[0].export_ledger(h)), to_oracle(engs[1].export_ledger(h)), f"h={h}")


def test_step_graph_reads_caller_buffers():
    """Flat serving path (bf16, d = 128): the captured step kernel is pointed at the caller's q / k /
    v (mpa_decode_step_rebind, no staging copy) and back at its own buffers for host-buffer steps;
    interleaving both gives the eager (graph-free) engine's outputs bit-for-bit across updates."""
    from paper_2506_13059_b200.engine import DecodeEngine

    tr = gen_synthetic(8, 1000, HeadLayout(8, 2, 128), 0.1, seed=8, decode_steps=60)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64,
                       tokens_per_centroid=8, seed=8)
    P = tr.prompt_len
    engs = []
    for graphs in (True, False):
        e = DecodeEngine(cfg, tr.layout, 2, tcap=tr.total_len + 8, dtype=torch.bfloat16, use_graphs=graphs)
        k = torch.as_tensor(tr.keys[:, :P]).cuda()[None].repeat(2, 1, 1, 1)
        v = torch.as_tensor(tr.values[:, :P]).cuda()[None].repeat(2, 1, 1, 1)
        e.write_tokens(k, v)
        e.prefill()
        engs.append(e)
    assert engs[0].fused_lookup_path()
    oh = torch.empty(2, 8, 128, dtype=torch.float32).pin_memory()
    n_upd = 0
    for t in range(60):
        q = torch.as_tensor(tr.queries[:, t]).float()[None].repeat(2, 1, 1).contiguous()
        kn = torch.as_tensor(tr.keys[:, P + t]).float()[None].repeat(2, 1, 1).contiguous()
        vn = torch.as_tensor(tr.values[:, P + t]).float()[None].repeat(2, 1, 1).contiguous()
        ref = engs[1].step(q.cuda(), kn.cuda(), vn.cuda()).clone()
        if t % 3 == 2:
            engs[0].step_host(q.pin_memory(), kn.pin_memory(), vn.pin_memory(), oh)
            torch.cuda.synchronize()
            got = oh.cuda()
        else:
            qd, kd, vd = q.cuda(), kn.cuda(), vn.cuda()  # fresh device tensors every step
            got = engs[0].step(qd, kd, vd).clone()
        assert torch.equal(ref, got), t
        n_upd += engs[0].last_update is not None
    assert n_upd >= 3
    assert engs[0]._graph_raw is not None
    for h in range(engs[0].L):
        _assert_same_ledger(to_oracle(engs[0].export_ledger(h)), to_oracle(engs[1].export_ledger(h)), f"h={h}")
