"""Host cost of the batched end-to-end step (DecodeEngine.step_host): per-call CPU time without
syncs, next to the device-timed e2e step (CUDA events, as bench.py measures it, L2 flushed before
each step), and the device time of its parts (host->device copies, step graph, device->host copy)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    args = argparse.Namespace(batch=16, ctx=32768, budget=512, steps=a.steps + 10, warmup=3, workload="c2")
    dev = torch.device("cuda", 0)
    eng, Q, KN, VN, _ = bench.build_engine(args, 0, dev)
    b, Hq, d = Q.shape[1], Q.shape[2], Q.shape[3]
    qh = Q.cpu().pin_memory()
    kh, vh = KN.cpu().pin_memory(), VN.cpu().pin_memory()
    oh = torch.empty(b, Hq, d, dtype=torch.float32).pin_memory()
    flush = bench.L2Flush(dev)
    for i in range(5):
        eng.step_host(qh[i], kh[i], vh[i], oh)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        return e

    tot, parts, host = [], [], []
    if os.environ.get("E2E_WARM_ALL"):  # touch every step's pinned slice once before timing
        for i in range(a.steps):
            eng.step_host(qh[5 + i], kh[5 + i], vh[5 + i], oh)
        torch.cuda.synchronize()
    for i in range(a.steps):
        flush(i)
        e0 = ev()
        t0 = time.perf_counter()
        eng.step_host(qh[5 + i], kh[5 + i], vh[5 + i], oh)
        host.append((time.perf_counter() - t0) * 1e6)
        e1 = ev()
        tot.append((e0, e1))
    torch.cuda.synchronize()
    # the parts, same order as step_host, each bracketed
    for i in range(a.steps):
        flush(i)
        e0 = ev()
        eng._gq.copy_(qh[5 + i], non_blocking=True)
        eng._gk.copy_(kh[5 + i][:, :, None], non_blocking=True)
        eng._gv.copy_(vh[5 + i][:, :, None], non_blocking=True)
        e1 = ev()
        eng._graph.replay()
        e2 = ev()
        oh.copy_(eng.out, non_blocking=True)
        e3 = ev()
        parts.append((e0, e1, e2, e3))
    torch.cuda.synchronize()
    med = lambda xs: sorted(xs)[len(xs) // 2]
    e2e = [x.elapsed_time(y) * 1e3 for x, y in tot]
    print(f"step_host: host {med(host):.1f} us median; device e0->e1 {med(e2e):.1f} us median, "
          f"{sum(e2e) / len(e2e):.1f} us mean, top {sorted(e2e)[-5:]}")
    print(f"parts: h2d {med([p[0].elapsed_time(p[1]) * 1e3 for p in parts]):.1f} us, graph "
          f"{med([p[1].elapsed_time(p[2]) * 1e3 for p in parts]):.1f} us, d2h {med([p[2].elapsed_time(p[3]) * 1e3 for p in parts]):.1f} us")


if __name__ == "__main__":
    main()
