#!/usr/bin/env python
"""Full-size BASELINE configs 1-5 on one B200 (measurement tool, not a test).

  python tools/run_config.py config3 [config4 ...] [--out gpurun_out/full_configs.json] [--phases]

Each run: generator (seeded, paper_2506_08355_b200/problems.py), explicit generalized nullspace
(Y0 = M^-1 X0 by the device CG), operators resident in HBM, then one warm-up-free solve through
the public API (bosp.solve) with eigenvectors copied back to host buffers.  Seconds from the
solver's CUDA events (device_s) and the host wall clock (solve_s).  Results are re-checked on the
host independently of the solver: unnormalised and normalised residuals of
H z = lambda z (bosp_solver.cpp:271,496), max|X^T Y - I| and its spectral norm,
ascending order, and the nullspace cross-Gram max|X0^T Y|.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


PROFILE_RANGE = False
REPEAT = 1


def make(name: str, bosp, P):
    if name == "config1":
        return P.config1()
    if name == "config2":
        return P.config2(64, solve=bosp.device_solver)
    if name == "config3":
        return P.config3(128, solve=bosp.device_solver)
    if name == "config4":
        return P.config4(solve_factory=bosp.device_solver)
    if name == "config5":
        return P.config5(1024, solve=bosp.device_solver)
    if name.startswith("config3@"):       # config3@64: same family, smaller grid
        return P.config3(int(name.split("@")[1]), solve=bosp.device_solver)
    raise SystemExit(f"unknown config {name}")


def host_apply(op, x, P):
    if isinstance(op, np.ndarray):
        return op @ x
    if isinstance(op, P.Stencil):
        op = op.to_csr()
    return op.scipy() @ x


def run(name: str) -> dict:
    from paper_2506_08355_b200 import bosp
    from paper_2506_08355_b200 import problems as P
    t0 = time.perf_counter()
    prob = make(name, bosp, P)
    gen_s = time.perf_counter() - t0
    K, M = bosp.operators_for(prob)
    cfg = bosp.BospConfig(**prob.cfg)
    ns = bosp.GeneralizedNullspace(prob.x0, prob.y0)
    bosp.device_sync()
    bosp.launch_reset()
    if PROFILE_RANGE:  # ncu --profile-from-start off sees exactly this solve
        bosp.lib().bosp_profiler_range(1)
    warm = []
    for _ in range(REPEAT - 1):  # extra solves (eigenvectors stay in HBM), then the checked one
        warm.append(bosp.solve(K, M, None, cfg, ns, want_vectors=False).stats["device_seconds"])
    t1 = time.perf_counter()
    res = bosp.solve(K, M, None, cfg, ns, want_vectors=True)
    solve_s = time.perf_counter() - t1
    if PROFILE_RANGE:
        bosp.lib().bosp_profiler_range(0)
    launches = bosp.launch_count()
    x, y, lam = res.x, res.y, res.lambdas
    # independent host checks (bosp_solver.cpp:256-271): K x = lambda y, M y = lambda x
    kx = host_apply(prob.K, x, P)
    my = host_apply(prob.M, y, P)
    r = np.sqrt(np.sum((kx - y * lam) ** 2, 0) + np.sum((my - x * lam) ** 2, 0))
    nz = np.sqrt(np.sum(x ** 2, 0) + np.sum(y ** 2, 0))
    raw = r / nz
    g = x.T @ y - np.eye(x.shape[1])
    return {
        "config": prob.name, "n": prob.n, "gen_s": gen_s, "solve_s": solve_s,
        "device_s": res.stats["device_seconds"], "iterations": res.iterations,
        "converged": res.converged, "nev_converged": res.nev_converged,
        "max_resid_normalized": float(np.max(raw / (1.0 + lam))), "max_resid_raw": float(raw.max()),
        "max_abs_XtY_minus_I": float(np.abs(g).max()),
        "spectral_XtY_minus_I": float(np.linalg.norm(g, 2)),
        "sorted": bool(np.all(np.diff(lam) >= 0)), "lambda_min": float(lam.min()),
        "lambda_max": float(lam.max()), "repairs": res.stats["repairs"],
        "cg_iterations": res.stats["cg_iterations"], "host_small_s": res.stats["host_small_seconds"],
        "launches": launches, "launch_families": bosp.launch_families(),
        "max_width_u": res.stats["max_width_u"],
        "nullspace_crossgram": float(np.abs(prob.x0.T @ y).max()),
        "eigenpairs_per_s": prob.cfg["nev"] / res.stats["device_seconds"],
        "device_s_all": warm + [res.stats["device_seconds"]],
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--out", default=None)
    ap.add_argument("--repeat", type=int, default=1, help="solves per config (the last one is checked)")
    ap.add_argument("--profile-range", action="store_true",
                    help="cudaProfilerStart/Stop around the solve (for ncu --profile-from-start off)")
    a = ap.parse_args()
    global PROFILE_RANGE, REPEAT
    PROFILE_RANGE = a.profile_range
    REPEAT = max(1, a.repeat)
    out = {}
    for c in a.configs:
        r = run(c)
        out[r["config"]] = r
        print(json.dumps(r), flush=True)
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
