import sys, os
sys.path.insert(0, '/root/repo')
from paper_1805_06124_b200 import inputs, rbg
S, w, tol, _ = inputs.config1(M=700, N=300)
for k_max in (1, 2, 3, 5, 10, 40):
    g = rbg.greedy(S, w, tol, k_max)
    print("k_max", k_max, "->", g.k, g.stop, flush=True)
