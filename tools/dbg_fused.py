import sys; sys.path.insert(0, '.')
import numpy as np, torch
sys.path.insert(0, 'tests')
from oracle import tensor_oracle as O
import test_tc_fused_gpu as t
O.build()
for case in [(5, 256, 512, 8, 2), (5, 4096, 14336, 8, 2), (2, 4096, 14336, 1, 1)]:
    hf, yf, h2, y2, hr, yr = t.run(O, *case, seed=case[0] + 3 * case[3])
    print(case, "h fused==2launch", np.array_equal(hf, h2), "h diff frac", (hf != h2).mean(),
          "y maxdiff fused-2l", float(np.abs(yf - y2).max()), "y fused-oracle", float(np.abs(yf - yr).max()),
          "y 2l-oracle", float(np.abs(y2 - yr).max()), "ymax", float(np.abs(yr).max()),
          "h fused!=oracle", (hf != hr).mean(), "h 2l!=oracle", (h2 != hr).mean())
