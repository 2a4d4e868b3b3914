import gc, sys, time, os
sys.path.insert(0, os.getcwd())
t0 = [0.0]
def cb(phase, info):
    if phase == "start":
        t0[0] = time.perf_counter()
    else:
        dt = (time.perf_counter() - t0[0]) * 1e3
        if dt > 1.0:
            print(f"GC gen {info['generation']} {dt:.1f} ms collected {info['collected']}", file=sys.stderr)
gc.callbacks.append(cb)
import bench
sys.argv = ["bench.py", "--workload", "c4", "--no-cpu"]
bench.main()
