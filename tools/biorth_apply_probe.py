#!/usr/bin/env python
"""ncu target: one fused MGS-Biorth application (P = X A, Q = Y B, P^T Q) at n rows, k = kb.

  python tools/biorth_apply_probe.py [n] [k]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_08355_b200 import bosp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 21
k = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rng = np.random.default_rng(1)
x = np.asfortranarray(rng.uniform(-1, 1, (n, k)))
y = np.asfortranarray(rng.uniform(-1, 1, (n, k)))
a = np.asfortranarray(np.triu(rng.uniform(-1, 1, (k, k))))
b = np.asfortranarray(np.triu(rng.uniform(-1, 1, (k, k))))
for _ in range(2):
    p, q, g = bosp._test_biorth_apply(x, y, a, b)
print("max |P^T Q - (XA)^T (YB)| =", float(np.abs(g - (x @ a).T @ (y @ b)).max()))
