import cProfile, pstats, sys, os, argparse
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2506_13059_b200 import clustering
args = argparse.Namespace(batch=16, ctx=32768, budget=512, steps=2, warmup=3, workload="c2")
eng, Q, KN, VN, _ = bench.build_engine(args, 0, torch.device("cuda", 0))
L = eng.cfg.local_buffer
need = int(2 * L - (eng.cache_len[0] - eng.buffer_start[0]))
eng.write_tokens(torch.randn(eng.n_seq, eng.Hkv, need, 128, device="cuda"), torch.randn(eng.n_seq, eng.Hkv, need, 128, device="cuda"))
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
clustering.online_update(eng, list(range(eng.n_seq)), 0)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
