"""Algorithmic byte counts of the decode path (the reference's vector-load
accounting, bench.py:53-71, converted to bytes).

Per ledger (sequence x kv-head), with S scored centroids, R rejected centroids, X exact tokens
(sinks + buffer + selected members), c bytes per cache element, G q-heads per kv-head:
    lookup (K9/K10): S * (d*c + 4)                   key centroids + sizes
    fused  (K11/12): X * (2*d*c + 4) + R * (d*c + 4*G + 4) + 2*G*d*4
                     exact K_rot/V rows + token ids, value centroids + reused logits + codes,
                     q in / out
    dense  (K13)   : 2 * n * d * c + 2*G*d*4
"""

from __future__ import annotations

import numpy as np


def decode_bytes(stats: np.ndarray, scored: np.ndarray, d: int, G: int, elem: int) -> dict:
    """stats: [L, 4] (n_tok, n_rej, sel_tokens, n_sel) from DecodeEngine.head_stats()."""
    X = stats[:, 0].astype(np.float64)
    R = stats[:, 1].astype(np.float64)
    S = np.asarray(scored, np.float64)
    lookup = float(np.sum(S * (d * elem + 4)))
    fused = float(np.sum(X * (2 * d * elem + 4) + R * (d * elem + 4 * G + 4) + 2 * G * d * 4))
    return {"lookup": lookup, "fused": fused, "step": lookup + fused}


def dense_bytes(cache_len: np.ndarray, d: int, G: int, elem: int) -> float:
    n = np.asarray(cache_len, np.float64)
    return float(np.sum(2 * n * d * elem + 2 * G * d * 4))
