"""One staged draw_stats launch (the bench's dominant kernel) for the ncu --set full traffic capture.

Prints the launch's algorithmic bytes (bench.py roofline: 4 B per staged word read, 148 B per
pre-drawn row, 2 B per tail value) so tools/traffic_json.py can relate the captured DRAM bytes.
Run under ncu with -k regex:draw_stats -s 1 -c 1 (the second call's launch).
"""
import json
import sys
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf

g = float(sys.argv[1]) if len(sys.argv) > 1 else 2.5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
R = int(sys.argv[3]) if len(sys.argv) > 3 else 400000  # one chunk at n = 1000
eng = engine.get_engine()
ks = torch.empty(R, dtype=torch.float64, device='cuda'); gh = torch.empty_like(ks); st = torch.empty(R, dtype=torch.uint8, device='cuda')
u = torch.empty(R * eng.staging_stride(n), dtype=torch.int32, device='cuda')
t = eng.table(g, None, lambda: sampling_cdf(g, Support(None)))
eng.stage_uniforms(1, 0, 0, R, n, u)
cnt = torch.zeros(13, dtype=torch.int64, device='cuda')
eng.set_counters(cnt)
eng.run_replicates_staged(t, None, g, n, 1, 0, 0, R, u, 0, R, ks, gh, st)
torch.cuda.synchronize()
eng.set_counters(None)
w = [int(x) for x in cnt.cpu().tolist()]
staged, rows, tails = w[8], w[11], w[12]
for _ in range(2):
    eng.run_replicates_staged(t, None, g, n, 1, 0, 0, R, u, 0, R, ks, gh, st)
torch.cuda.synchronize()
print(json.dumps({"gamma": g, "n": n, "rows": rows, "staged_words": staged, "tail_values": tails,
                  "algorithmic_bytes": 4 * staged + 148 * rows + 2 * tails}))
