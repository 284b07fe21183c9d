"""Prints how the walk outputs of tests/walk_accel_case.py differ between two runs (npz files)."""
import sys

import numpy as np

a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for k in a.files:
    if k.endswith("_steps"):
        print(k, int(a[k][0]), int(b[k][0]), "rel diff %.2e" % (abs(int(a[k][0]) - int(b[k][0])) / int(a[k][0])))
    else:
        d = np.abs(a[k] - b[k])
        print(k, "close %.4f" % np.mean(d <= 1e-5 * np.abs(a[k]).max()), "max diff %.3e" % d.max(), "changed", int(np.sum(d > 0)), "of", d.size)
