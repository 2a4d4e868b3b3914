"""Generate golden fixtures by running the REAL reference package.

Run in the build container only (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz.  tests/test_golden_oracle.py checks that the oracle
restatement (oracle/mpa_oracle.py) reproduces every array bit-for-bit; the GPU
parity tests then use the pinned oracle as their checker.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from multipole_attn import attention as A  # noqa: E402
from multipole_attn import clustering as C  # noqa: E402
from multipole_attn import pipeline as P  # noqa: E402
from multipole_attn.core import EngineConfig, HeadLayout, HierarchyConfig, gen_synthetic  # noqa: E402
from multipole_attn.rope import RopeParams, rotate  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def ref_ledger_arrays(led, prefix: str, out: dict) -> None:
    blocks = led.sealed + [led.final]
    out[prefix + "meta"] = np.array([led.sink_end, led.buffer_start, led.total, led.split_count, len(blocks)], np.int64)
    out[prefix + "spans"] = np.array([[b.start, b.end] for b in blocks], np.int64).reshape(-1, 2)
    for lv, get in (("fine", lambda b: b.clusters), ("coarse", lambda b: b.level1)):
        levs = [get(b) for b in blocks]
        if any(x is None for x in levs):
            continue
        cl = [c for x in levs for c in x]
        d = blocks[0].clusters[0].key_centroid.shape[0] if blocks[0].clusters else 0
        out[prefix + lv + "_counts"] = np.array([len(x) for x in levs], np.int64)
        out[prefix + lv + "_sizes"] = np.array([c.size for c in cl], np.int64)
        out[prefix + lv + "_members"] = np.concatenate([c.member_indices for c in cl]).astype(np.int64) if cl else np.zeros(0, np.int64)
        out[prefix + lv + "_kc"] = np.stack([c.key_centroid for c in cl]) if cl else np.zeros((0, d))
        out[prefix + lv + "_vc"] = np.stack([c.value_centroid for c in cl]) if cl else np.zeros((0, d))
        if lv == "coarse":
            kids = [np.asarray(c.children, np.int64) for c in cl]
            out[prefix + "coarse_children"] = np.concatenate(kids) if kids else np.zeros(0, np.int64)


def refs_array(refs) -> np.ndarray:
    return np.array(refs, np.int64).reshape(-1, 3)


# ---------------------------------------------------------------------------


def case_rope(out):
    rng = np.random.default_rng(100)
    v = rng.standard_normal((7, 16)).astype(np.float32)
    pos = np.array([0, 1, 63, 4096, 131071, 65535, 777])
    out["rope_v"] = v
    out["rope_pos"] = pos
    for th in (1e4, 1e6):
        out[f"rope_out_{int(th)}"] = rotate(v, pos, RopeParams(16, th))
    v128 = rng.standard_normal((5, 128)).astype(np.float32)
    out["rope_v128"] = v128
    out["rope_out128"] = rotate(v128, np.array([0, 17, 32768, 65536, 131071]), RopeParams(128, 1e6))


def case_synthetic(out):
    tr = gen_synthetic(8, 600, HeadLayout(8, 2, 16), 0.05, seed=11, decode_steps=20)
    out["syn_small_keys"], out["syn_small_values"], out["syn_small_queries"] = tr.keys, tr.values, tr.queries
    big = gen_synthetic(256, 8192, HeadLayout(32, 8, 128), 0.05, seed=0, decode_steps=32)
    out["syn_c1_sha"] = np.array([sha(big.keys), sha(big.values), sha(big.queries)])


def _mixture(n, d, k, seed, sigma=0.05):
    rng = np.random.default_rng(seed)
    means = rng.standard_normal((k, d))
    means /= np.linalg.norm(means, axis=1, keepdims=True)
    labels = rng.integers(0, k, size=n)
    return means[labels] + sigma * rng.standard_normal((n, d))


def case_kmeans(out):
    cases = [(_mixture(300, 8, 6, s), 6, 5, s) for s in range(4)]
    cases += [(np.zeros((20, 4)), 4, 3, 1), (np.eye(3), 10, 3, 0), (_mixture(400, 8, 8, 5), 16, 10, 2)]
    for i, (pts, k, it, seed) in enumerate(cases):
        cl = C.kmeans(pts, k, it, seed)
        out[f"km{i}_pts"] = pts
        out[f"km{i}_args"] = np.array([k, it, seed])
        out[f"km{i}_kc"] = np.stack([c.key_centroid for c in cl])
        out[f"km{i}_sizes"] = np.array([c.size for c in cl])
        out[f"km{i}_members"] = np.concatenate([c.member_indices for c in cl])


def _ledger_cfg(hier=None):
    return EngineConfig(block_size=128, alpha=64, local_buffer=16, sink_tokens=8, token_budget=32,
                        tokens_per_centroid=8, hierarchy=hier, seed=5)


def case_ledgers(out):
    tr = gen_synthetic(6, 500, HeadLayout(2, 2, 8), 0.05, seed=5, decode_steps=200)
    for tag, hier in (("flat", None), ("hier", HierarchyConfig(32, 8, 0.5))):
        cfg = _ledger_cfg(hier)
        for h in range(2):
            led = C.build_prefill_index_head(tr.keys[h, :500], tr.values[h, :500], 500, cfg, h)
            ref_ledger_arrays(led, f"led_{tag}_h{h}_prefill_", out)
        # sliding updates on head 0 until two splits happened (test_clustering.py:179-194)
        keys, values = tr.keys[0], tr.values[0]
        led = C.build_prefill_index_head(keys[:500], values[:500], 500, cfg, head=0)
        n, u = 500, 0
        while led.split_count < 2 and n + 16 <= keys.shape[0]:
            n += 16
            led.total = n
            C.append_tokens(led, keys[:n], values[:n], cfg, np.random.default_rng(n), head=0)
            ref_ledger_arrays(led, f"led_{tag}_upd{u}_", out)
            u += 1
        out[f"led_{tag}_nupd"] = np.array(u)


def case_lookups(out):
    lay = HeadLayout(1, 1, 8)
    tr = gen_synthetic(6, 400, lay, 0.05, seed=10, decode_steps=0)
    for tag, hier in (("flat", None), ("hp3", HierarchyConfig(32, 8, 0.3)), ("hp1", HierarchyConfig(32, 8, 1.0))):
        cfg = EngineConfig(block_size=128, alpha=64, local_buffer=16, sink_tokens=8, token_budget=48,
                           tokens_per_centroid=8, hierarchy=hier, seed=10)
        led = C.build_prefill_index_head(tr.keys[0], tr.values[0], 400, cfg, head=0)
        ref_ledger_arrays(led, f"lk_{tag}_led_", out)
        rng = np.random.default_rng(77)
        for qi in range(6):
            G = 1 if qi < 3 else 4
            q = rng.standard_normal((G, 8)) * (1.0 + 2.0 * qi)
            fn = A.flat_lookup if hier is None else A.hierarchical_lookup
            sel_idx, sel_refs, frej, crej, stats = fn(q, led, cfg, 8)
            p = f"lk_{tag}_q{qi}_"
            out[p + "q"] = q
            out[p + "sel_idx"] = sel_idx
            out[p + "sel_refs"] = refs_array(sel_refs)
            out[p + "frej_refs"] = refs_array([r for r, _, _ in frej])
            out[p + "frej_logits"] = np.array([lg for _, _, lg in frej]).reshape(-1, G)
            out[p + "crej_refs"] = refs_array([r for r, _, _ in crej])
            out[p + "crej_logits"] = np.array([lg for _, _, lg in crej]).reshape(-1, G)
            out[p + "stats"] = np.array([stats["scored_centroids"], stats["rejected_centroids"]])


def _record_run(out, prefix, reports):
    out[prefix + "outputs"] = np.stack([r.outputs for r in reports])
    out[prefix + "updates"] = np.array([r.update_occurred for r in reports])
    if reports[0].per_head:
        out[prefix + "stats"] = np.array([[[h.selected_tokens, h.scored_centroids, h.rejected_centroids]
                                           for h in r.per_head] for r in reports])
        out[prefix + "buffer_len"] = np.array([r.buffer_len for r in reports])
        sel = [s for r in reports for s in r.selected_indices]
        out[prefix + "sel_counts"] = np.array([s.size for s in sel])
        out[prefix + "sel_concat"] = np.concatenate(sel) if sel else np.zeros(0, np.int64)


def case_runs(out):
    lay = HeadLayout(8, 2, 16)
    small = gen_synthetic(8, 600, lay, 0.05, seed=11, decode_steps=20)
    cfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64, seed=11)
    for mode in P.MODES:
        n = 6 if mode == "oracle" else 20
        _record_run(out, f"run_small_{mode}_", P.run(small, cfg, mode=mode, max_steps=n, collect_outputs=True))
    full = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=10**6, seed=11)
    _record_run(out, "run_small_fullbudget_", P.run(small, full, max_steps=6, collect_outputs=True))
    tr = gen_synthetic(8, 600, lay, 0.05, seed=13, decode_steps=40)
    hcfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64,
                        hierarchy=HierarchyConfig(32, 8, 0.5), seed=13)
    _record_run(out, "run_hier_", P.run(tr, hcfg, max_steps=40, collect_outputs=True))
    # long online-update trajectory with several splits (C4 analogue at desk scale)
    lt = gen_synthetic(8, 1000, HeadLayout(4, 1, 16), 0.1, seed=3, decode_steps=400)
    lcfg = EngineConfig(block_size=256, alpha=128, local_buffer=16, sink_tokens=5, token_budget=64, seed=3)
    st = P.prefill(lt, lcfg)
    reps = []
    for t in range(lt.decode_steps):
        pos = lt.prompt_len + t
        o, r = P.step(st, lt.queries[:, t], lt.keys[:, pos], lt.values[:, pos])
        r.outputs = o
        reps.append(r)
    _record_run(out, "run_long_", reps)
    ref_ledger_arrays(st.ledgers[0], "run_long_final_led_", out)


def case_c1(out):
    lay = HeadLayout(32, 8, 128)
    tr = gen_synthetic(256, 8192, lay, 0.05, seed=0, decode_steps=32)
    cfg = EngineConfig(tokens_per_centroid=32, token_budget=819, seed=0)
    st = P.prefill(tr, cfg)
    for h, led in enumerate(st.ledgers):
        blk = led.final
        out[f"c1_h{h}_sizes"] = np.array([c.size for c in blk.clusters], np.int32)
        out[f"c1_h{h}_members"] = np.concatenate([c.member_indices for c in blk.clusters]).astype(np.int32)
        out[f"c1_h{h}_kc_sha"] = np.array(sha(np.stack([c.key_centroid for c in blk.clusters])))
        out[f"c1_h{h}_vc_sha"] = np.array(sha(np.stack([c.value_centroid for c in blk.clusters])))
    reps = []
    for t in range(3):
        pos = tr.prompt_len + t
        o, r = P.step(st, tr.queries[:, t], tr.keys[:, pos], tr.values[:, pos])
        r.outputs = o
        reps.append(r)
    _record_run(out, "c1_", reps)


def main():
    for name, fn in (("rope", case_rope), ("synthetic", case_synthetic), ("kmeans", case_kmeans),
                     ("ledgers", case_ledgers), ("lookups", case_lookups), ("runs", case_runs), ("c1", case_c1)):
        out = {}
        fn(out)
        np.savez_compressed(os.path.join(OUT, f"golden_{name}.npz"), **out)
        print(name, len(out), "arrays")


if __name__ == "__main__":
    main()
