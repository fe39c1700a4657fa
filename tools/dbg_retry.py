import sys
sys.path.insert(0, '.')
import numpy as np
from oracle import port
sys.path.insert(0, 'tests')
from test_gpu_parity import run_cell
for K, g, n in [(6, -20.0, 140), (8, -20.0, 128), (8, -22.0, 60)]:
    ks, gh, st = run_cell(K, g, n, 7, 0, 0, 48)
    for j in range(48):
        try:
            w = port.replicate(g, K, n, 7, j, 0)
        except port.FailedTwice:
            w = (None, None, 2)
        if st[j] != w[2] or (w[0] is not None and abs(ks[j] - w[0]) > 1e-9 * abs(w[0]) + 1e-12):
            print(K, g, n, j, "got", st[j], ks[j], gh[j], "want", w)
