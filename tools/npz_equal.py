"""Compare two .npz dumps array by array (bit equality). Usage: python tools/npz_equal.py a.npz b.npz"""
import sys

import numpy as np

a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
bad = 0
for k in a.files:
    if not np.array_equal(a[k], b[k]):
        bad += 1
        print(k, "max|diff|", np.abs(a[k] - b[k]).max(), "max|a|", np.abs(a[k]).max())
print("mismatching", bad, "of", len(a.files))
