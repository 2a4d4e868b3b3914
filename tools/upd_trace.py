"""Online-update events at the bench workload (C2, batch 16): per-phase wall time
(MPA_UPD_TRACE) and per-kernel device time from the CUDA profiler (CUPTI), steady-state
events only (the first event pays lazy module loads)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MPA_UPD_TRACE"] = "1"


def main():
    import torch

    import bench
    from paper_2506_13059_b200 import clustering

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--events", type=int, default=2)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--workload", default="c2")
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
        upd = clustering.online_update(eng, list(range(eng.n_seq)), eng.cursor + ev)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3, upd

    ms, upd = event(0)
    print(f"event 0 (cold) {ms:.2f} ms {upd}", flush=True)
    from torch.profiler import ProfilerActivity, profile

    tot = 0.0
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for ev in range(1, a.events + 1):
            ms, upd = event(ev)
            tot += ms
            print(f"event {ev} {ms:.2f} ms {upd}", flush=True)
    print(f"mean {tot / a.events:.2f} ms/event")
    rows = []
    for e in prof.key_averages():
        t = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
        if t > 0:
            rows.append((t / a.events / 1e3, e.count // a.events, e.key[:70]))
    rows.sort(reverse=True)
    print(f"{'ms/event':>9} {'n/event':>8}  kernel")
    for t, n, k in rows[:25]:
        print(f"{t:9.3f} {n:8d}  {k}")
    print(f"{sum(r[0] for r in rows):9.3f}           total device")
    # per-launch durations (us) of the main kernels, in launch order, last event
    seq = {}
    for e in prof.events():
        if e.device_type.name == "CUDA" and e.name.startswith(("mpa::km_", "void mpa::km_")):
            nm = e.name.split("(")[0].replace("void ", "").replace("mpa::", "")
            seq.setdefault(nm, []).append(round(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total, 1))
    for nm, v in seq.items():
        if len(v) > 2:
            half = v[len(v) // a.events * (a.events - 1):]
            print(f"{nm:32s} {half}")
    # the last event's device timeline: busy time vs the gaps between consecutive kernels
    ks = sorted((e.time_range.start, e.time_range.end) for e in prof.events()
                if e.device_type.name == "CUDA" and e.name.startswith(("mpa::km_", "void mpa::km_")))
    ks = ks[len(ks) // a.events * (a.events - 1):]
    gaps = [b[0] - a_[1] for a_, b in zip(ks, ks[1:])]
    small = [g for g in gaps if 0 < g < 50]
    print(f"last event: {len(ks)} kernels, span {(ks[-1][1] - ks[0][0]) / 1e3:.2f} ms, busy "
          f"{sum(e - s for s, e in ks) / 1e3:.2f} ms, gaps <50us {sum(small) / 1e3:.2f} ms over {len(small)} "
          f"(median {sorted(small)[len(small) // 2] if small else 0:.1f} us), gaps >=50us "
          f"{sum(g for g in gaps if g >= 50) / 1e3:.2f} ms over {sum(1 for g in gaps if g >= 50)}")


if __name__ == "__main__":
    main()
