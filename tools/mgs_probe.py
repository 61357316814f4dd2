#!/usr/bin/env python
"""MGS-Biorth at HBM scale, one call = pair Gram + coefficients + fused application + check Gram
(the solver's dev_mgs_biorth), timed with CUDA events; then one profiled call split by launch
family.

  python tools/mgs_probe.py [n] [m] [--reps R]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_08355_b200 import bosp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("n", nargs="?", type=int, default=2 ** 21)
    ap.add_argument("m", nargs="?", type=int, default=20)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    byts = 48.0 * a.n * a.m
    for kind in ("mgs", "mgs_cold"):
        ms = bosp.bench_blas(kind, a.n, a.m, a.m, reps=a.reps)
        print(f"{kind:8s} n={a.n} m={a.m}: {ms * 1e3:.1f} us/call, {byts / ms / 1e6:.1f} GB/s (48 n m bytes)")
    bosp.profile_enable("*")
    bosp.bench_blas("mgs", a.n, a.m, a.m, reps=3)
    rep = bosp.profile_collect()
    bosp.profile_enable(None)
    for f, v in sorted(rep["families"].items(), key=lambda kv: -kv[1]["ms"]):
        print(f"  {f:14s} {v['launches']:4d} launches {v['ms'] * 1e3 / max(1, v['launches']):8.1f} us/launch")


if __name__ == "__main__":
    main()
