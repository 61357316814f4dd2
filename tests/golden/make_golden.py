"""Generate the committed golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run here (needs /root/reference to build oracle/_ref):  python tests/golden/make_golden.py [--big]
Outputs (small, committed):
  tests/golden/golden_small.npz   RNG stream, kernel KATs on seeded inputs, T(s) solves
  tests/golden/golden_solves.json eigenvalues / residuals / iterations of the reference on the
                                  paper tables and BASELINE configs 1 (and 2 with --big)
Every input is regenerated from a seed by the tests, so only outputs are stored.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2506_08355_b200 import problems as P  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# PAPER.md:1782-1791 (Table 3, Advanpix quadruple-precision column) -- published pins for
# K = T(-1), M = T(0), n = 1000.
TABLE3_ADVANPIX = [3.943890108210e-05, 6.154958719056e-05, 1.577542931907e-04,
                   1.994584196853e-04, 3.549418750556e-04, 4.161478616511e-04,
                   6.309942290978e-04, 7.116221744879e-04, 9.859008227908e-04,
                   1.085870497647e-03]


def kernel_inputs(seed: int, n: int, m: int):
    """Seeded inputs shared by make_golden and the tests."""
    rng = np.random.default_rng(seed)
    return (np.asfortranarray(rng.uniform(-1, 1, (n, m))),
            np.asfortranarray(rng.uniform(-1, 1, (n, m))))


def small_fixtures():
    g = {}
    g["rng_seed0"] = ref.fill_uniform(0, 2000)
    g["rng_seed12345"] = ref.fill_uniform(12345, 777)
    # block kernels
    x, y = kernel_inputs(1, 300, 7)
    g["inner_xy"] = ref.block_inner(x, y)
    c = np.asfortranarray(np.random.default_rng(2).uniform(-1, 1, (7, 5)))
    g["product_xc"] = ref.block_product(x, c)
    g["axpy_yxc"] = ref.block_axpy(x, c, y[:, :5])
    # MGS / CGS biorth
    for tag, seed, n, m in (("a", 3, 200, 12), ("b", 4, 64, 30)):
        x, y = kernel_inputs(seed, n, m)
        p, q, kept, dropped = ref.mgs_biorth(x, y)
        g[f"mgs_{tag}_p"], g[f"mgs_{tag}_q"] = p, q
        g[f"mgs_{tag}_kept"] = np.array(kept)
        g[f"mgs_{tag}_res"] = np.array([ref.biorth_residual(p, q)])
    # biorth_against with two bases
    x, y = kernel_inputs(5, 150, 6)
    bx, by = kernel_inputs(6, 150, 4)
    bp, bq, _, _ = ref.mgs_biorth(bx, by)
    cx, cy = kernel_inputs(7, 150, 3)
    cp, cq, _, _ = ref.mgs_biorth(cx, cy)
    g["against_w"], g["against_z"] = ref.biorth_against([(bp, bq), (cp, cq)], x, y)
    # CG on T(0) n=50, 4 rhs, loose and tight
    t = P.t_matrix(50, 0.0)
    rhs = np.asfortranarray(np.random.default_rng(8).uniform(-1, 1, (50, 4)))
    for tol, it in ((1e-2, 20), (1e-12, 100)):
        xx, br, mi = ref.cg_solve(t.spec(), rhs, tol=tol, max_iter=it)
        g[f"cg_{it}"] = xx
        g[f"cg_{it}_maxit"] = np.array([mi])
    # small LREP on a random SPD pair d=12 (k=5)
    rng = np.random.default_rng(9)
    a = rng.standard_normal((12, 12)); kh = a @ a.T + 12 * np.eye(12)
    b = rng.standard_normal((12, 12)); mh = b @ b.T + 12 * np.eye(12)
    g["small_k"], g["small_m"] = kh, mh
    g["small_lam"], g["small_xhat"], g["small_yhat"] = ref.solve_small_lrep(kh, mh, 5)
    u, s, v, sweeps, conv = ref.jacobi_svd(a)
    g["svd_sigma"] = s
    return g


def solve_record(prob_k, prob_m, cfg, ns, n, label):
    t0 = time.time()
    r = ref.solve(prob_k, prob_m, cfg, ns=ns, want_vectors=False)
    dt = time.time() - t0
    print(f"{label}: {dt:.2f}s iters={r.stats['iterations']} converged={r.stats['converged']}",
          flush=True)
    return dict(lambdas=[float(v) for v in r.lambdas], residuals=[float(v) for v in r.residuals],
                iterations=int(r.stats["iterations"]), converged=bool(r.stats["converged"]),
                nev_converged=int(r.stats["nev_converged"]),
                final_biorth_deviation=float(r.stats["final_biorth_deviation"]),
                max_width_u=int(r.stats["max_width_u"]), seconds=dt, threads=ref.threads(),
                cfg=dict(nev=cfg.nev, nb=cfg.nb, tol=cfg.tol, moving=cfg.moving, seed=cfg.rng_seed))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also run config 2 at 64^3 (~6 min)")
    ap.add_argument("--c3", action="store_true", help="also run the config-3 family at 20^3, nev 100 (~90 s)")
    ap.add_argument("--only-c3", action="store_true", help="only (re)run the config-3 family entry")
    args = ap.parse_args()
    if args.only_c3:
        path = os.path.join(OUT, "golden_solves.json")
        solves = json.load(open(path))
        p = P.config3(20)
        solves["config3_m20"] = solve_record(p.oracle_spec("K"), p.oracle_spec("M"), ref.RefConfig(**p.cfg), (p.x0, p.y0), p.n, "config3 m=20 nev=100")
        json.dump(solves, open(path, "w"), indent=1)
        return
    ref.set_threads(0)
    np.savez_compressed(os.path.join(OUT, "golden_small.npz"), **small_fixtures())

    path = os.path.join(OUT, "golden_solves.json")
    solves = json.load(open(path)) if os.path.exists(path) else {}
    solves["_source"] = "oracle/_ref (unmodified reference, -O3 -DNDEBUG -fopenmp) via tests/golden/make_golden.py"
    solves["table3_advanpix"] = dict(lambdas=TABLE3_ADVANPIX, source="PAPER.md:1782-1791")
    for n in (100, 1000):
        t = P.t_matrix(n, 0.0)
        solves[f"t0_t0_n{n}"] = solve_record(t.spec(), t.spec(), ref.RefConfig(nev=10 if n == 1000 else 5, nb=10 if n == 1000 else 5, tol=1e-10), None, n, f"T0/T0 n={n}")
    for n in (100, 1000):
        tm, t0 = P.t_matrix(n, -1.0), P.t_matrix(n, 0.0)
        solves[f"tm1_t0_n{n}"] = solve_record(tm.spec(), t0.spec(), ref.RefConfig(nev=10 if n == 1000 else 5, nb=10 if n == 1000 else 5, tol=1e-10), P.analytic_nullspace_T(n), n, f"T-1/T0 n={n}")
    # odd sizes for the row-partition tests (ragged slices)
    for n, k in ((300, 4), (401, 5)):
        tm, t0 = P.t_matrix(n, -1.0), P.t_matrix(n, 0.0)
        solves[f"tm1_t0_n{n}"] = solve_record(tm.spec(), t0.spec(), ref.RefConfig(nev=k, nb=k, tol=1e-10), P.analytic_nullspace_T(n), n, f"T-1/T0 n={n}")
    # moving-mechanism case on T(0): nev=12, nb=2 -> moving on, locks happen
    t = P.t_matrix(400, 0.0)
    solves["t0_moving_n400"] = solve_record(t.spec(), t.spec(), ref.RefConfig(nev=12, nb=2, tol=1e-9), None, 400, "T0 moving")
    # small grid versions of configs 2 and 5 (oracle-fast)
    for m in (8, 16):
        p = P.config2(m)
        solves[f"config2_m{m}"] = solve_record(p.oracle_spec("K"), p.oracle_spec("M"), ref.RefConfig(nev=20, nb=40, tol=1e-8), (p.x0, p.y0), p.n, f"config2 m={m}")
    p = P.config5(32)
    solves["config5_m32"] = solve_record(p.oracle_spec("K"), p.oracle_spec("M"), ref.RefConfig(nev=40, nb=8, tol=1e-8), (p.x0, p.y0), p.n, "config5 m=32 nev=40 nb=8")
    p = P.config1()
    solves["config1"] = solve_record(p.oracle_spec("K"), p.oracle_spec("M"), ref.RefConfig(**p.cfg), (p.x0, p.y0), p.n, "config1")
    if args.c3:
        p = P.config3(20)
        solves["config3_m20"] = solve_record(p.oracle_spec("K"), p.oracle_spec("M"), ref.RefConfig(**p.cfg), (p.x0, p.y0), p.n, "config3 m=20 nev=100")
    if args.big:
        p = P.config2(64)
        solves["config2"] = solve_record(p.oracle_spec("K"), p.oracle_spec("M"), ref.RefConfig(**p.cfg), (p.x0, p.y0), p.n, "config2 64^3")
    json.dump(solves, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
