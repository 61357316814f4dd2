"""Golden eigenvalues for BASELINE configs 3, 4 and 5 *as configured* (nev / nb / moving exactly
as BASELINE.json states them) at sizes the UNMODIFIED reference (oracle/_ref) finishes here.

Run here (needs oracle/_ref):   python tests/golden/make_golden_configs.py config4 [--threads T]
Each config writes its own file tests/golden/golden_<name>.json (so several can run at once):
  config4_n4096  dense BSE-like, K = Pi(A-B)Pi with a 64-dim null basis, nev 32, nb 64 (-> 32)
  config5_m64    5-point 64^2 grid, nev 500, nb 64, moving (3+ locking events), d = 320
  config3_m32    7-point 32^3 grid, nev 100, nb 64, moving=true, d = 320
The inputs are regenerated from seeds by tests/test_gpu_configs.py (problems.py), so only the
reference's outputs are stored.  SURVEY.md section 8(d): reduced sizes of the same families.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2506_08355_b200 import problems as P  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

def _mass_1d(n):
    """Linear-FEM mass matrix h/6 [1 4 1] with h = 1: a sparse SPD weight B."""
    import numpy as np
    import scipy.sparse as sp
    e = np.ones(n)
    return P.csr_from_scipy(sp.diags([e[:-1] / 6, 4 * e / 6, e[:-1] / 6], [-1, 0, 1]))


def weighted_case(n):
    """K = M = T(0), inner product weighted by the sparse mass matrix B: (K x = lambda B y,
    M y = lambda B x), nev 6, nb 6, tol 1e-10 -- the reference detects the (empty) nullspace."""
    t = P.t_matrix(n, 0.0)
    return dict(K=t, M=t, B=_mass_1d(n), n=n, cfg=dict(nev=6, nb=6, tol=1e-10), name=f"weighted-T0-massB-n{n}")


CASES = {
    "weighted_massB_n400": lambda: weighted_case(400),
    "weighted_massB_n2000": lambda: weighted_case(2000),
    "config4_n4096": lambda: P.config4(n=4096),
    "config5_m64": lambda: P.config5(64),
    "config3_m32": lambda: P.config3(32),
}


def run(name: str):
    p = CASES[name]()
    if isinstance(p, dict):  # B-weighted case: operators as CSR, nullspace detected by the reference
        cfg = ref.RefConfig(**p["cfg"])
        t0 = time.time()
        r = ref.solve(p["K"].spec(), p["M"].spec(), cfg, B=p["B"].spec(), want_vectors=False)
        dt = time.time() - t0
        p = type("W", (), {"name": p["name"], "n": p["n"]})
    else:
        cfg = ref.RefConfig(**p.cfg)
        t0 = time.time()
        r = ref.solve(p.oracle_spec("K"), p.oracle_spec("M"), cfg, ns=(p.x0, p.y0), want_vectors=False)
        dt = time.time() - t0
    rec = dict(lambdas=[float(v) for v in r.lambdas], residuals=[float(v) for v in r.residuals],
               iterations=int(r.stats["iterations"]), converged=bool(r.stats["converged"]),
               nev_converged=int(r.stats["nev_converged"]),
               final_biorth_deviation=float(r.stats["final_biorth_deviation"]),
               max_width_u=int(r.stats["max_width_u"]), seconds=dt, threads=ref.threads(),
               problem=p.name, n=p.n,
               cfg=dict(nev=cfg.nev, nb=cfg.nb, tol=cfg.tol, moving=cfg.moving, seed=cfg.rng_seed),
               _source="oracle/_ref (unmodified reference, -O3 -DNDEBUG -fopenmp) via "
                       "tests/golden/make_golden_configs.py")
    print(f"{name}: {dt:.1f}s iters={rec['iterations']} converged={rec['converged']}", flush=True)
    with open(os.path.join(OUT, f"golden_{name}.json"), "w") as f:
        json.dump(rec, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+", choices=sorted(CASES))
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    ref.set_threads(a.threads)
    for n in a.names:
        run(n)


if __name__ == "__main__":
    main()
