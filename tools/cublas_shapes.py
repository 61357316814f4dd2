#!/usr/bin/env python
"""cuBLAS DGEMM (torch fp64 matmul) on the solver's tall-skinny shapes next to the library's own
DMMA kernels on the same shapes (bosp_bench_blas): the in-solve roofline reference.

  python tools/cublas_shapes.py [n]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_08355_b200 import bosp  # noqa: E402


def t_cublas(f, reps=10):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 21
    dev = torch.device("cuda")
    for kind, a, b in (("gram", 320, 320), ("gram", 64, 320), ("product", 320, 192), ("product", 320, 320),
                       ("product", 320, 64)):
        x = torch.randn(a, n, dtype=torch.float64, device=dev)   # column-major n x a == row-major a x n
        y = torch.randn(b if kind == "gram" else a, n if kind == "gram" else b, dtype=torch.float64, device=dev)
        if kind == "gram":      # G = X^T Y (a x b) over n rows
            ms = t_cublas(lambda: torch.mm(x, y.t()))
            flops = 2.0 * n * a * b
        else:                   # Out (n x b) = X (n x a) C (a x b)
            c = torch.randn(b, a, dtype=torch.float64, device=dev)
            ms = t_cublas(lambda: torch.mm(c, x))
            flops = 2.0 * n * a * b
        own = bosp.bench_blas(kind, n, a, b, reps=10)
        print(f"{kind:8s} {a}x{b} n={n}: cuBLAS {ms:8.3f} ms {flops / ms / 1e9:6.2f} TF/s | "
              f"B200 kernels {own:8.3f} ms {flops / own / 1e9:6.2f} TF/s", flush=True)
        del x, y


if __name__ == "__main__":
    main()
