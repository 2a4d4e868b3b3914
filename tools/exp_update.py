"""Time one online-update event at the bench workload, phase by phase (host wall clock with
device syncs), plus the GPU kernel time of each phase via CUDA events."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    from paper_2506_13059_b200 import clustering

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=32768)
    a = ap.parse_args()
    args = argparse.Namespace(batch=a.batch, ctx=a.ctx, budget=512, steps=2, warmup=3)
    eng, Q, KN, VN, _ = bench.build_engine(args, 0, torch.device("cuda", 0))
    L = eng.cfg.local_buffer
    gen = torch.Generator(device="cuda").manual_seed(5)
    need = int(2 * L - (eng.cache_len[0] - eng.buffer_start[0]))
    eng.write_tokens(torch.randn(eng.n_seq, eng.Hkv, need, 128, generator=gen, device="cuda"),
                     torch.randn(eng.n_seq, eng.Hkv, need, 128, generator=gen, device="cuda"))
    torch.cuda.synchronize()
    orig = {name: getattr(clustering, name) for name in ("_write_fine", "_refresh_counts", "_split", "_hierarchy")}
    times = {}

    def wrap(name, fn):
        def w(*x, **k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fn(*x, **k)
            torch.cuda.synchronize()
            times[name] = times.get(name, 0.0) + time.perf_counter() - t0
            return r
        return w

    for name, fn in orig.items():
        setattr(clustering, name, wrap(name, fn))
    KM = clustering.KMeansBatch
    orig_lloyd = KM.lloyd

    def lloyd(self):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = orig_lloyd(self)
        torch.cuda.synchronize()
        times["lloyd"] = times.get("lloyd", 0.0) + time.perf_counter() - t0
        times["lloyd_rounds"] = r
        return r

    KM.lloyd = lloyd
    t0 = time.perf_counter()
    upd = clustering.online_update(eng, list(range(eng.n_seq)), 0)
    torch.cuda.synchronize()
    total = time.perf_counter() - t0
    print("update total ms", round(total * 1e3, 2), upd)
    for k, v in times.items():
        print(f"  {k:16s} {v * 1e3 if k != 'lloyd_rounds' else v:9.2f}")


def recheck_stats():
    """Rows re-scored in fp64 by the last tcgen05 assignment pass of a Lloyd call."""
    import torch

    from paper_2506_13059_b200 import clustering

    orig = clustering.KMeansBatch.lloyd

    def lloyd(self):
        r = orig(self)
        if self.tc_ws is not None:
            kpad = (self.sum_k + 255) // 256 * 256 + 256
            o = 3 * kpad * self.d * 2
            o = (o + 255) & ~255
            o += kpad * 4
            o = (o + 255) & ~255
            o += self.P * 8
            o = (o + 255) & ~255
            o += self.sum_n * 8
            cnt = int(self.tc_ws[o:o + 4].view(torch.int32).item())
            print(f"  recheck rows (last pass): {cnt} of {self.sum_n}")
        return r

    clustering.KMeansBatch.lloyd = lloyd


def call_stats():
    """Per C-ABI call wall time (device-synchronised) inside one update."""
    import collections

    import torch

    from paper_2506_13059_b200 import clustering

    orig = clustering.call
    tot = collections.defaultdict(float)

    def call(name, *a):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = orig(name, *a)
        torch.cuda.synchronize()
        tot[name] += time.perf_counter() - t0
        return r

    clustering.call = call
    orig_init = clustering.KMeansBatch.__init__

    def init(self, *a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        orig_init(self, *a, **k)
        torch.cuda.synchronize()
        tot["KMeansBatch.__init__"] += time.perf_counter() - t0

    clustering.KMeansBatch.__init__ = init
    import atexit

    atexit.register(lambda: [print(f"  call {k:28s} {v * 1e3:8.2f} ms") for k, v in sorted(tot.items(), key=lambda x: -x[1])])


def steady_state():
    """Wall time of eng.step around an update in steady state (after a first update), and of
    the graph recapture that follows it."""
    import torch

    import bench

    args = argparse.Namespace(batch=8, ctx=16384, budget=512, steps=300, warmup=3)
    eng, Q, KN, VN, _ = bench.build_engine(args, 0, torch.device("cuda", 0))
    L = eng.cfg.local_buffer
    t_up, t_other = [], []
    for i in range(3 * L + 10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.step(Q[i % Q.shape[0]], KN[i % KN.shape[0]], VN[i % VN.shape[0]])
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        (t_up if eng.last_update is not None else t_other).append(dt)
    g0 = time.perf_counter()
    eng.invalidate_graph()
    eng._capture_step()
    torch.cuda.synchronize()
    print(f"steps {len(t_other)} median {np.median(t_other) * 1e6:.1f} us; update steps {[round(x * 1e3, 2) for x in t_up]} ms;"
          f" recapture {(time.perf_counter() - g0) * 1e3:.2f} ms")


if __name__ == "__main__":
    if os.environ.get("RECHECK"):
        recheck_stats()
    if os.environ.get("CALLS"):
        call_stats()
    if os.environ.get("STEADY"):
        steady_state()
    else:
        main()
