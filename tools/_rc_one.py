"""One resampling event at N (default 2^22) on normal log-weights, 3 calls (ncu target)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
lw = np.random.default_rng(0).normal(0, 1, n)
for _ in range(3):
    capi.systematic_resample(lw, 0.37)
