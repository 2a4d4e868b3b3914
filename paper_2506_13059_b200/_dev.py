"""numpy <-> device glue for the reference-API modules (rope.py, attention.py, the module-level
clustering functions): uploads the caller's arrays, runs the fp64 kernels of csrc/mpa_refapi.cu
through the C ABI, and returns numpy results.  There is no CPU fallback: without a CUDA device or
libmpattn.so every call raises."""

from __future__ import annotations

import numpy as np
import torch

from ._lib import call, lib, ptr, stream_ptr


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the multipole_attn API runs on the B200 kernels: no CUDA device (there is no CPU fallback)")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def f64(a) -> torch.Tensor:
    return torch.tensor(np.asarray(a, dtype=np.float64), device=device())  # a copy: inputs may be read-only views


def i64(a) -> torch.Tensor:
    return torch.tensor(np.asarray(a, dtype=np.int64), device=device())


def rotate(x: np.ndarray, pos: np.ndarray, inv_freq: np.ndarray) -> np.ndarray:
    n, d = x.shape
    xt, pt, ft = f64(x), f64(pos), f64(inv_freq)
    out = torch.empty_like(xt)
    call("mpa_ref_rotate", ptr(xt), ptr(pt), n, d, ptr(ft), ptr(out), stream_ptr())
    return out.cpu().numpy()


def logits(q: np.ndarray, x: np.ndarray) -> np.ndarray:
    """[G, n] = q[G, d] . x[n, d]^T / sqrt(d)."""
    q = np.atleast_2d(q)
    G, d = q.shape
    n = x.shape[0]
    out = torch.empty(G, max(n, 1), dtype=torch.float64, device=device())
    if n:
        qt, xt = f64(q), f64(x)
        call("mpa_ref_logits", ptr(qt), ptr(xt), G, n, d, ptr(out), stream_ptr())
    return out[:, :n].cpu().numpy()


def partial(lg: np.ndarray, values: np.ndarray, weights: np.ndarray | None = None, want_weights: bool = False):
    """(a, m, s[, normalised weights]) of the streaming softmax over n >= 1 logits."""
    n, d = values.shape
    lt, vt = f64(lg), f64(values)
    wt = f64(weights) if weights is not None else None
    out = torch.empty(d + 2, dtype=torch.float64, device=device())
    wo = torch.empty(n, dtype=torch.float64, device=device()) if want_weights else None
    call("mpa_ref_partial", ptr(lt), ptr(vt), ptr(wt), n, d, ptr(out), ptr(wo), stream_ptr())
    o = out.cpu().numpy()
    res = (o[:d].copy(), float(o[d]), float(o[d + 1]))
    return res + (wo.cpu().numpy(),) if want_weights else res


def group_scores(lg: np.ndarray, sizes: np.ndarray) -> np.ndarray:
    """mean over the G rows of e / (e . sizes), e = exp(l - row max)."""
    G, n = lg.shape
    lt, st = f64(lg), f64(sizes)
    sc = torch.empty(n, dtype=torch.float64, device=device())
    call("mpa_ref_group_scores", ptr(lt), ptr(st), G, n, ptr(sc), None, stream_ptr())
    return sc.cpu().numpy()


def nearest(points: np.ndarray, centroids: np.ndarray) -> np.ndarray:
    n, d = points.shape
    k = centroids.shape[0]
    out = torch.empty(max(n, 1), dtype=torch.int64, device=device())
    if n:
        pt, ct = f64(points), f64(centroids)
        call("mpa_ref_nearest", ptr(pt), ptr(ct), n, k, d, ptr(out), stream_ptr())
    return out[:n].cpu().numpy()


def seg_stats(points: np.ndarray, members: list, centroids: np.ndarray | None = None,
              weights: np.ndarray | None = None):
    """Per cluster (member index arrays into the rows of points): in-order means [k, d] (size-weighted
    with `weights` per point row) and, with centroids, the total squared error about them."""
    k = len(members)
    d = points.shape[1]
    off = np.zeros(k + 1, np.int64)
    np.cumsum([len(m) for m in members], out=off[1:])
    idx = np.concatenate([np.asarray(m, np.int64) for m in members]) if k else np.zeros(0, np.int64)
    pt, ot, it = f64(points), i64(off), i64(idx if idx.size else np.zeros(1, np.int64))
    mean = torch.empty(max(k, 1), d, dtype=torch.float64, device=device())
    ct = f64(centroids) if centroids is not None else None
    sq = torch.zeros(1, dtype=torch.float64, device=device())
    wt = f64(weights) if weights is not None else None
    call("mpa_ref_seg_stats", ptr(pt), ptr(ot), ptr(it), ptr(wt), k, d, ptr(mean), ptr(ct),
         ptr(sq) if ct is not None else None, stream_ptr())
    return mean[:k].cpu().numpy(), float(sq.item())
