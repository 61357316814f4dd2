#!/usr/bin/env python
"""Operator apply / batched-CG microbenchmark on device-resident data (measurement tool).

  python tools/apply_probe.py [config3|config5|config2] [--cols 64,20] [--reps 20]

Prints mean ms per apply (bosp_bench_apply) and per batched CG iteration with all columns active
(bosp_bench_cg), and the stored-format HBM bytes / s of the apply (16 n m for the stencils).
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="config3")
    ap.add_argument("--cols", default="64,20")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    from paper_2506_08355_b200 import bosp
    from paper_2506_08355_b200 import problems as P
    import numpy as np
    dense = lambda n: (None, np.asfortranarray(np.random.default_rng(1).standard_normal((n, n))))
    kop, mop = {"config4": lambda: dense(16384), "config1": lambda: dense(2000), "config3": lambda: P._grid3_ops(128), "config2": lambda: (P.config2(64).K, P.config2(64).M),
                "config5": lambda: (P.Stencil(1024, 1024, 1, "neumann", 1.0),
                                    P.Stencil(1024, 1024, 1, "dirichlet", 1.0, "array", v=[1.5] * (1024 * 1024)))}[a.config]()
    if isinstance(mop, np.ndarray):
        M = bosp.LinearOperator.from_dense(mop)
    elif isinstance(mop, P.Stencil):
        M = bosp.LinearOperator.from_stencil(mop)
    else:
        M = bosp.LinearOperator.from_csr(mop)
    n = M.dim
    for m in (int(c) for c in a.cols.split(",")):
        ms = bosp.bench_apply(M, m, reps=a.reps)
        cg = bosp.bench_cg(M, m, iters=20, reps=3)
        extra = f" {2.0 * n * n * m / ms / 1e9:6.2f} TF/s (dense)" if isinstance(mop, np.ndarray) else ""
        print(f"{a.config} n={n} m={m}: apply {ms * 1e3:8.1f} us ({16.0 * n * m / ms / 1e6:7.1f} GB/s){extra}  "
              f"cg iteration {cg * 1e3:8.1f} us", flush=True)


if __name__ == "__main__":
    main()
