import sys; sys.path.insert(0,'.')
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf
eng = engine.get_engine()
for K,g,n in [(None,2.5,100),(None,2.5,2000),(1000,0.5,100),(20,1.0,1000),(2,1.0,10),(None,2.0,100000),(5000,1.5,500)]:
    for R in (1, 64, 5000):
        ks = torch.empty(R, dtype=torch.float64, device='cuda'); gh=torch.empty_like(ks); st=torch.empty(R,dtype=torch.uint8,device='cuda')
        t = eng.table(g, K, lambda: sampling_cdf(g, Support(K)))
        try:
            eng.run_replicates(t, K, g, n, 1, 0, 0, R, ks, gh, st); torch.cuda.synchronize()
            print("ok", K, g, n, R, float(ks[0]))
        except Exception as e:
            print("FAIL", K, g, n, R, e)
