"""Where does the public-API sweep spend host time?  (diagnostic)"""
import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import torch
import paper_1305_6738_b200 as zk
from paper_1305_6738_b200.engine import get_engine
import bench
eng = get_engine()
R = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
sup = zk.Support.unbounded()
zk.build_table(bench.NS, bench.GAMMAS, sup, base_seed=1, replicates=R, repetitions=1)
torch.cuda.synchronize()
for clear in (False, True):
    if clear:
        eng.clear_tables()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pr = cProfile.Profile(); pr.enable()
    zk.build_table(bench.NS, bench.GAMMAS, sup, base_seed=1, replicates=R, repetitions=1)
    pr.disable()
    print("clear", clear, "seconds", time.perf_counter() - t0)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
