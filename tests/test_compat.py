"""Source-level drop-in: reference callers compile unchanged against the B200 build.

Two callers, both written against the reference's public headers (proj/include/bosp/...):
  * oracle/ref_shim.cpp -- the C shim this repo uses to drive the UNMODIFIED reference
    (oracle/Makefile).  It touches ~50 names of the reference API (solve, initialize /
    iterate_once with SolverState fields, LinearOperator factories, biorth, block kernels,
    cg_solve, the small LREP, nullspace, Matrix Market, the exception classes).
  * tests/compat/ref_api_usage.cpp -- a standalone program in the reference's idiom
    (size_t sizes, std::span columns, csr_from_triplets, an ApplyFn callback).
CPU tests: both compile against include/bosp/* (forwarding to paper_2506_08355_b200/csrc/api.hpp)
and link libbosp_b200.so; the usage program also compiles against the reference headers
themselves when /root/reference is present (this container).  GPU tests: the compat-built
shim runs through oracle/ref.py's own wrappers -- i.e. the reference's caller, unmodified, on
the B200 -- and must reproduce the reference's golden results; the usage binary runs too.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2506_08355_b200")
OUT = os.path.join(PKG, "csrc", "build")
SHIM_SRC = os.path.join(ROOT, "oracle", "ref_shim.cpp")
USAGE_SRC = os.path.join(ROOT, "tests", "compat", "ref_api_usage.cpp")
SHIM_SO = os.path.join(OUT, "ref_shim_b200.so")
USAGE_BIN = os.path.join(OUT, "ref_api_usage_b200")
REF_INCLUDE = "/root/reference/proj/include"
B200_FLAGS = ["-std=c++20", "-O1", "-Wall", "-Wno-sign-compare", "-I", os.path.join(ROOT, "include"),
              "-I", os.path.join(PKG, "csrc"), "-I", "/usr/local/cuda/include"]
LINK = ["-L" + PKG, "-lbosp_b200", "-Wl,-rpath," + PKG]


def _gxx(args):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    r = subprocess.run(["g++", *args], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return r


def _lib_built():
    if not os.path.exists(os.path.join(PKG, "libbosp_b200.so")):
        pytest.fail("libbosp_b200.so not built: run __graft_entry__.build()")


def build_shim():
    _lib_built()
    os.makedirs(OUT, exist_ok=True)
    _gxx([*B200_FLAGS, "-fPIC", "-shared", SHIM_SRC, *LINK, "-o", SHIM_SO])
    return SHIM_SO


def build_usage():
    _lib_built()
    os.makedirs(OUT, exist_ok=True)
    _gxx([*B200_FLAGS, USAGE_SRC, *LINK, "-o", USAGE_BIN])
    return USAGE_BIN


def test_reference_shim_compiles_unchanged_against_b200():
    so = build_shim()
    nm = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    src = open(SHIM_SRC).read()
    import re
    wanted = set(re.findall(r"^int (ref_[a-z_0-9]+)\(", src, flags=re.M))
    assert len(wanted) >= 15
    missing = [w for w in wanted if f" T {w}" not in nm]
    assert not missing, missing
    # every bosp:: symbol the shim needs resolves inside libbosp_b200 (mangled b200 names)
    und = subprocess.run(["nm", "-D", "--undefined-only", so], capture_output=True, text=True).stdout
    assert "bosp4b200" in und


def test_reference_style_program_compiles_against_both():
    if os.path.isdir(REF_INCLUDE):  # the caller is genuine reference-API code
        _gxx(["-std=c++20", "-fsyntax-only", "-I", REF_INCLUDE, USAGE_SRC])
    assert os.path.exists(build_usage())


# ---- on the GPU: the reference's caller, unmodified, driving the B200 build ---------------

@pytest.fixture()
def ref_on_b200():
    from oracle import ref
    ref.use_library(build_shim())
    try:
        yield ref
    finally:
        ref.use_library(None)


@pytest.mark.gpu
def test_usage_program_runs_on_b200():
    binary = build_usage()
    r = subprocess.run([binary], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "lambda_max_rel_err" in r.stdout


@pytest.mark.gpu
def test_reference_shim_solves_on_b200(ref_on_b200, golden_solves):
    ref = ref_on_b200
    from paper_2506_08355_b200 import problems as P
    n = 1000
    km, t0 = P.t_matrix(n, -1.0), P.t_matrix(n, 0.0)
    r = ref.solve(km.spec(), t0.spec(), ref.RefConfig(nev=10, nb=10, tol=1e-10), ns=P.analytic_nullspace_T(n))
    g = golden_solves["tm1_t0_n1000"]["lambdas"]
    assert r.stats["converged"]
    assert np.abs(r.lambdas - g).max() / np.abs(g).max() < 1e-10
    assert r.residuals.max() < 1e-10
    assert np.abs(r.x.T @ r.y - np.eye(10)).max() < 1e-10
    p = P.config2(16)
    r2 = ref.solve(p.oracle_spec("K"), p.oracle_spec("M"), ref.RefConfig(nev=20, nb=40, tol=1e-8), ns=(p.x0, p.y0))
    g2 = np.asarray(golden_solves["config2_m16"]["lambdas"])
    assert np.abs(r2.lambdas - g2).max() / g2.max() < 1e-10


@pytest.mark.gpu
def test_reference_shim_kernels_on_b200(ref_on_b200, golden_small):
    """The shim's kernel-level entry points (mgs_biorth, block_inner, cg_solve, small LREP,
    iterate_once via time_iterations) against the reference's golden fixtures."""
    ref = ref_on_b200
    from tests.golden.make_golden import kernel_inputs
    from paper_2506_08355_b200 import problems as P
    x, y = kernel_inputs(1, 300, 7)
    assert np.allclose(ref.block_inner(x, y), golden_small["inner_xy"], rtol=1e-13, atol=1e-13)
    x, y = kernel_inputs(3, 200, 12)
    p, q, kept, _ = ref.mgs_biorth(x, y)
    assert list(kept) == list(golden_small["mgs_a_kept"])
    assert np.allclose(p, golden_small["mgs_a_p"], rtol=1e-9, atol=1e-9)
    lam, xh, yh = ref.solve_small_lrep(golden_small["small_k"], golden_small["small_m"], 5)
    assert np.allclose(lam, golden_small["small_lam"], rtol=1e-13)
    t = P.t_matrix(50, 0.0)
    rhs = np.asfortranarray(np.random.default_rng(8).uniform(-1, 1, (50, 4)))
    xx, _, _ = ref.cg_solve(t.spec(), rhs, tol=1e-12, max_iter=100)
    assert np.allclose(xx, golden_small["cg_100"], rtol=1e-10, atol=1e-12)
    n = 300
    tm = P.t_matrix(n, -1.0)
    out = ref.time_iterations(tm.spec(), P.t_matrix(n, 0.0).spec(), ref.RefConfig(nev=4, nb=4, tol=1e-10),
                              P.analytic_nullspace_T(n), 100)
    assert out["converged"] and out["nev_conv"] >= 4
