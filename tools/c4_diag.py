"""bench.py --workload c4 with every Python GC pause over 1 ms logged to stderr (with MPA_UPD_TRACE=1
the online updates log their phases too): separates interpreter pauses from device-side stalls.
python tools/c4_diag.py"""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

_t0 = [0.0]


def _gc_timer(phase, info):
    if phase == "start":
        _t0[0] = time.perf_counter()
    else:
        dt = (time.perf_counter() - _t0[0]) * 1e3
        if dt > 1.0:
            print(f"GC gen {info['generation']} {dt:.1f} ms collected {info['collected']}", file=sys.stderr)


def main():
    import bench

    gc.callbacks.append(_gc_timer)
    sys.argv = ["bench.py", "--workload", "c4", "--no-cpu"]
    bench.main()


if __name__ == "__main__":
    main()
