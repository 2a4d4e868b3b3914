"""A/B of the dense decode (mpa_sparse_decode with tok == NULL) at C2 b16 32K: flat engine, random
tokens, cold L2 per launch, CUDA events.  MPATTN_LIB selects the library under test."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    from paper_2506_13059_b200.core import EngineConfig, HeadLayout
    from paper_2506_13059_b200.engine import DecodeEngine

    lay = HeadLayout(32, 8, 128)
    cfg = EngineConfig(tokens_per_centroid=16, rope_theta=1e6)
    b, ctx = 16, 32768
    dev = torch.device("cuda", 0)
    eng = DecodeEngine(cfg, lay, b, tcap=ctx + 64, dtype=torch.bfloat16)
    g = torch.Generator(device=dev).manual_seed(1)
    for s in range(b):
        k = torch.randn(1, 8, ctx, 128, generator=g, device=dev)
        bench._write_seq(eng, s, k, k)
    eng.cache_len[:] = ctx
    eng._sync_scalars()
    eng.ntok_dense_d.fill_(ctx)
    q = torch.randn(b, 32, 128, generator=g, device=dev)
    fl = bench.L2Flush(dev)
    ts = []
    for i in range(25):
        fl(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.attend_dense(q)
        e1.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(os.environ.get("MPATTN_LIB", "current"), "dense us median", round(ts[len(ts) // 2], 1), "min", round(ts[0], 1))


if __name__ == "__main__":
    main()
