#!/usr/bin/env python
"""Tall-skinny fp64 kernels on device-resident random data (measurement / ncu target).

  python tools/blas_probe.py [n] [--reps R] [--shapes gram:320x320,product:320x192,...]

Prints mean ms and TFLOP/s (or GB/s) per call from the library's own CUDA-event microbenchmark
(bosp_bench_blas).  Under ncu, use small --reps and -k regex:k_gram / k_product.
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("n", nargs="?", type=int, default=128 ** 3)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--shapes", default="gram:320x320,product:320x192,product:320x64,gram:20x20,gram3:20x20,gramsym:20x20,gram3:64x64,gramsym:64x64,gramsym:320x320")
    a = ap.parse_args()
    from paper_2506_08355_b200 import bosp
    for item in a.shapes.split(","):
        kind, dims = item.split(":")
        x, y = (int(v) for v in dims.split("x"))
        ms = bosp.bench_blas(kind, a.n, x, y, reps=a.reps)
        flops = 2.0 * a.n * x * y * (3 if kind in ("gram3", "gramsym") else 1)
        byts = 8.0 * a.n * (x + y) + (8.0 * a.n * y if kind == "axpy" else 0.0)
        if kind == "mgs":  # X, Y read + P, Q written + the P^T Q check = 48 n m
            flops, byts = 6.0 * a.n * x * x, 48.0 * a.n * x
        elif kind == "mgsapply":
            flops, byts = 6.0 * a.n * x * x, 32.0 * a.n * x
        print(f"{kind:8s} n={a.n} {x}x{y}: {ms * 1e3:9.1f} us  {flops / ms / 1e9:7.2f} TF/s  "
              f"{byts / ms / 1e6:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
