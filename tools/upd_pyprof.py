"""Host-side profile of online-update events (cProfile, no per-phase syncs): where the Python
time of an event goes, next to its wall time."""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    from paper_2506_13059_b200 import clustering

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--ctx", type=int, default=16384)
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--events", type=int, default=2)
    a = ap.parse_args()
    args = argparse.Namespace(batch=a.batch, ctx=a.ctx, budget=512, steps=2, warmup=3, workload=a.workload)
    dev = torch.device("cuda", 0)
    eng, Q, KN, VN, _ = bench.build_engine(args, 0, dev)
    L = eng.cfg.local_buffer
    gen = torch.Generator(device="cuda").manual_seed(5)

    def event(ev):
        need = int(2 * L - (eng.cache_len[0] - eng.buffer_start[0]))
        if need > 0:
            eng.write_tokens(torch.randn(eng.n_seq, eng.Hkv, need, 128, generator=gen, device=dev),
                             torch.randn(eng.n_seq, eng.Hkv, need, 128, generator=gen, device=dev))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        clustering.online_update(eng, list(range(eng.n_seq)), eng.cursor + ev)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3

    event(0)
    walls = []
    pr = cProfile.Profile()
    for ev in range(1, a.events + 1):
        pr.enable()
        walls.append(event(ev))
        pr.disable()
    print("event wall ms:", [round(w, 2) for w in walls])
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(30)
    st.sort_stats("cumulative").print_stats(40)


if __name__ == "__main__":
    main()
