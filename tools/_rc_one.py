import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
from paper_2408_12057_b200 import capi
lw = np.random.default_rng(0).normal(0, 1, 1 << 22)
for _ in range(3):
    capi.systematic_resample(lw, 0.37)
