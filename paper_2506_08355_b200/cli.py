"""Command-line front end: `python -m paper_2506_08355_b200.cli solve ...` (SPEC.md cmd_solve,
/root/reference/SPEC.md:491-498 -- the reference ships no CLI source; this is the SURVEY 8(f)3
"Matrix Market + CLI/JSON report" row).

  solve --problem t0|tm1 --n N | --problem config1..config5 [--grid G]
        | --k-file K.mtx --m-file M.mtx [--b-file B.mtx]
        [--nev 10] [--nb ...] [--tol 1e-8] [--ngs 1] [--s 3] [--moving|--no-moving]
        [--max-iter 500] [--seed 0] [--rank-hint R] [--out report.json] [--history hist.csv]

Prints the eigenvalue table, writes a RunReport as canonical JSON (sorted keys; floats in
Python's shortest round-trip form, so parse + re-serialise is byte-identical and every value is
the exact real64) and the residual history as CSV (one row per iteration x tracked pair).
Exit codes (SPEC): 0 converged, 1 argument error, 2 ingestion error, 3 not converged (report
still written), 4 numerical abort.  Every solve runs on the B200 through libbosp_b200.so.
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

EXIT_OK, EXIT_PARSE, EXIT_INGEST, EXIT_NOTCONV, EXIT_ABORT = 0, 1, 2, 3, 4


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse exits 2 by default; the SPEC reserves 2 for ingestion
        self.print_usage(sys.stderr)
        print(f"error: {message}", file=sys.stderr)
        raise SystemExit(EXIT_PARSE)


def build_parser():
    ap = _Parser(prog="bosp", description="BOSP LREP eigensolver on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="solve an LREP and write a report")
    s.error = ap.error  # same exit code for subcommand argument errors
    s.add_argument("--problem", choices=["t0", "tm1", "config1", "config2", "config3", "config4", "config5"])
    s.add_argument("--n", type=int, default=None, help="T(s) size / dense config size")
    s.add_argument("--grid", type=int, default=None, help="grid points per axis (configs 2, 3, 5)")
    s.add_argument("--k-file")
    s.add_argument("--m-file")
    s.add_argument("--b-file")
    s.add_argument("--nev", type=int, default=None)
    s.add_argument("--nb", type=int, default=0)
    s.add_argument("--tol", type=float, default=1e-8)
    s.add_argument("--ngs", type=int, default=1)
    s.add_argument("--s", type=int, default=3)
    mv = s.add_mutually_exclusive_group()
    mv.add_argument("--moving", dest="moving", action="store_true", default=None)
    mv.add_argument("--no-moving", dest="moving", action="store_false")
    s.add_argument("--max-iter", type=int, default=500)
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--rank-hint", type=int, default=None)
    s.add_argument("--out", default=None)
    s.add_argument("--history", default=None)
    return ap


def _problem(a, bosp, P):
    """-> (K, M, B or None, nullspace or None, descriptor dict, default config dict)."""
    files = [a.k_file, a.m_file]
    if a.problem and any(files):
        raise ValueError("exactly one problem source: --problem or --k-file/--m-file")
    if not a.problem and not all(files):
        raise ValueError("exactly one problem source: --problem or --k-file/--m-file")
    if not a.problem:
        try:
            kc, mc = bosp.read_matrix_market(a.k_file), bosp.read_matrix_market(a.m_file)
            bc = bosp.read_matrix_market(a.b_file) if a.b_file else None
        except bosp.IngestionError:
            raise
        for c, f in ((kc, a.k_file), (mc, a.m_file), (bc, a.b_file)):
            if c is not None and not isinstance(c, P.Csr):
                raise bosp.IngestionError(f"{f}: operator must be square")
        if kc.n != mc.n or (bc is not None and bc.n != kc.n):
            raise bosp.IngestionError("K, M (and B) must have the same dimension")
        K, M = bosp.LinearOperator.from_csr(kc), bosp.LinearOperator.from_csr(mc)
        B = bosp.LinearOperator.from_csr(bc) if bc is not None else None
        return K, M, B, None, {"source": "matrix-market", "k_file": a.k_file, "m_file": a.m_file,
                               "b_file": a.b_file, "n": kc.n}, {}
    if a.problem in ("t0", "tm1"):
        n = a.n or 1000
        s = 0.0 if a.problem == "t0" else -1.0
        K = bosp.LinearOperator.from_csr(P.t_matrix(n, s))
        M = bosp.LinearOperator.from_csr(P.t_matrix(n, 0.0))
        ns = bosp.GeneralizedNullspace(*P.analytic_nullspace_T(n)) if a.problem == "tm1" else None
        return K, M, None, ns, {"source": "problem", "name": a.problem, "n": n}, {}
    gen = {"config1": lambda: P.config1(n=a.n or 2000),
           "config2": lambda: P.config2(a.grid or 64, solve=bosp.device_solver),
           "config3": lambda: P.config3(a.grid or 128, solve=bosp.device_solver),
           "config4": lambda: P.config4(n=a.n or 16384, solve_factory=bosp.device_solver),
           "config5": lambda: P.config5(a.grid or 1024, solve=bosp.device_solver)}[a.problem]
    p = gen()
    K, M = bosp.operators_for(p)
    return K, M, None, bosp.GeneralizedNullspace(p.x0, p.y0), {"source": "problem", "name": p.name,
                                                                  "n": p.n}, dict(p.cfg)


def cmd_solve(a) -> int:
    from . import bosp
    from . import problems as P
    try:
        K, M, B, ns, desc, dflt = _problem(a, bosp, P)
    except bosp.IngestionError as e:
        print(f"ingestion error: {e}", file=sys.stderr)
        return EXIT_INGEST
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INGEST if isinstance(e, OSError) else EXIT_PARSE
    cfgd = dict(dflt)
    for key, val in (("nev", a.nev), ("tol", a.tol), ("ngs", a.ngs), ("s", a.s), ("moving", a.moving),
                     ("max_outer_iter", a.max_iter), ("rng_seed", a.seed), ("rank_hint", a.rank_hint)):
        if val is not None:
            cfgd[key] = val
    if a.nb:
        cfgd["nb"] = a.nb
    cfgd.setdefault("nev", 10)
    cfg = bosp.BospConfig(**cfgd)
    t0 = time.perf_counter()
    try:
        res = bosp.solve(K, M, bosp.InnerProduct(B) if B is not None else None, cfg, ns, want_vectors=False)
    except bosp.NumericalAbort as e:
        print(f"numerical abort: {e}", file=sys.stderr)
        return EXIT_ABORT
    except bosp.ContractViolation as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_PARSE
    wall = time.perf_counter() - t0
    hist = np.asarray(res.history, dtype=float).reshape(-1, cfg.nev) if len(res.history) else np.zeros((0, cfg.nev))
    regression = []
    for j in range(cfg.nev):
        try:
            al, be, deg = bosp.regression_coefficients(hist, j, cfg.tol)
            regression.append({"pair": j, "alpha": al, "beta": be, "degenerate": bool(deg)})
        except bosp.BospError:
            regression.append({"pair": j, "alpha": None, "beta": None, "degenerate": None})
    report = {
        "config": {"nev": cfg.nev, "nb": cfg.effective_nb(), "tol": cfg.tol, "ngs": cfg.ngs, "s": cfg.s,
                   "moving": cfg.effective_moving(), "max_outer_iter": cfg.max_outer_iter,
                   "rng_seed": cfg.rng_seed, "rank_hint": cfg.rank_hint},
        "problem": desc,
        "eigenvalues": [float(v) for v in res.lambdas],
        "residuals": [float(v) for v in res.residuals],
        "iterations": int(res.iterations),
        "wall_seconds": wall,
        "device_seconds": float(res.stats["device_seconds"]),
        "converged": bool(res.converged),
        "nev_converged": int(res.nev_converged),
        "history": [[float(v) for v in row] for row in hist],
        "regression": regression,
    }
    print(f"{'pair':>4s} {'eigenvalue':>22s} {'residual':>12s}")
    for j, (lam, r) in enumerate(zip(res.lambdas, res.residuals)):
        print(f"{j + 1:4d} {lam:22.12E} {r:12.3E}")
    print(f"iterations {res.iterations}, converged {res.converged}, {wall:.3f} s")
    if a.out:
        with open(a.out, "w") as f:
            f.write(dumps(report))
    if a.history:
        with open(a.history, "w") as f:
            f.write("iteration,pair,residual\n")
            for it, row in enumerate(hist):
                for j, v in enumerate(row):
                    f.write(f"{it + 1},{j + 1},{float(v)!r}\n")
    return EXIT_OK if res.converged else EXIT_NOTCONV


def dumps(report) -> str:
    """Canonical JSON: sorted keys, floats as Python's shortest round-trip repr (real64-exact)."""
    return json.dumps(report, sort_keys=True, separators=(",", ":"), allow_nan=False) + "\n"


def main(argv=None) -> int:
    a = build_parser().parse_args(argv)
    if a.cmd == "solve":
        return cmd_solve(a)
    return EXIT_PARSE


if __name__ == "__main__":
    sys.exit(main())
