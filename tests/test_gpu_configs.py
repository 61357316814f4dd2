"""Oracle parity for BASELINE configs 3, 4 and 5 *as configured* (nev, nb, moving exactly as
BASELINE.json states them) at reduced sizes of the same families, against goldens produced by
the unmodified reference (tests/golden/make_golden_configs.py -> golden_config*.json).

  config4_n4096  dense BSE-like K = Pi(A-B)Pi (64-dim null), nev 32, nb 64 -> 32; the dense
                 K X / M Y path on the DMMA pipe (linear_operator.cpp:12-31)
  config5_m64    5-point 64^2 grid, nev 500, nb 64: moving with repeated locking
                 (bosp_solver.cpp:396-419), d = 320, deflation against the locked bases
  config3_m32    7-point 32^3 stencil, nev 100, nb 64, moving=true (matrix-free stencil kernel)

Bar (north_star): eigenvalues within 1e-10 relative of the reference, normalized residuals below
tol, max |X^T Y - I| < 1e-10.  Also: the device matrix-free plugin (bosp_op_device_callback)
solving the config-2 family, and a full-size config-3 self-consistency run (1 rank vs 2 ranks).
"""
import json
import os

import numpy as np
import pytest

from paper_2506_08355_b200 import bosp
from paper_2506_08355_b200 import problems as P
from tests.test_gpu_solver import check_result

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    path = os.path.join(GOLDEN, f"golden_{name}.json")
    if not os.path.exists(path):
        pytest.fail(f"missing reference golden {path} (tests/golden/make_golden_configs.py)")
    return json.load(open(path))


def solve_problem(p, cfg=None):
    K, M = bosp.operators_for(p)
    return bosp.solve(K, M, None, cfg or bosp.BospConfig(**p.cfg), bosp.GeneralizedNullspace(p.x0, p.y0))


def check_config(res, g, nev):
    assert g["converged"] and g["nev_converged"] == nev
    check_result(res, g["lambdas"], g["cfg"]["tol"], nev)
    # nullspace never leaks into the computed pairs
    return res


def test_config4_dense_bse_n4096():
    g = golden("config4_n4096")
    p = P.config4(n=4096)
    cfg = bosp.BospConfig(**p.cfg)
    assert cfg.effective_nb() == 32 and not cfg.effective_moving()
    res = check_config(solve_problem(p, cfg), g, 32)
    # K x = lambda M^-1 ... : the 64-dim nullspace stays deflated
    assert np.abs(p.y0.T @ res.x).max() < 1e-8 and np.abs(p.x0.T @ res.y).max() < 1e-8


def test_config5_as_configured_m64():
    g = golden("config5_m64")
    p = P.config5(64)
    cfg = bosp.BospConfig(**p.cfg)
    assert cfg.nev == 500 and cfg.effective_nb() == 64 and cfg.effective_moving()
    res = check_config(solve_problem(p, cfg), g, 500)
    assert res.stats["max_width_u"] <= g["max_width_u"] + 64


def test_config3_as_configured_m32():
    g = golden("config3_m32")
    p = P.config3(32)
    cfg = bosp.BospConfig(**p.cfg)
    assert cfg.nev == 100 and cfg.effective_nb() == 64 and cfg.effective_moving()
    check_config(solve_problem(p, cfg), g, 100)


def test_config3_csr_equals_stencil_m32():
    """The same config-3 problem through the CSR path (DIA/SELL kernels) and the matrix-free
    stencil: both meet the reference's eigenvalues."""
    g = golden("config3_m32")
    p = P.config3(32)
    K, M = (bosp.LinearOperator.from_csr(op.to_csr()) for op in (p.K, p.M))
    res = bosp.solve(K, M, None, bosp.BospConfig(**p.cfg), bosp.GeneralizedNullspace(p.x0, p.y0))
    check_config(res, g, 100)


# ---- device matrix-free plugin ------------------------------------------------------------

def _torch_csr_callback(csr, calls):
    """A user plugin: y = A x with torch's CSR SpMM on the solver's stream (device pointers
    wrapped through __cuda_array_interface__, nothing staged through the host)."""
    import torch
    a = torch.sparse_csr_tensor(torch.from_numpy(csr.rowptr), torch.from_numpy(csr.colidx),
                                torch.from_numpy(csr.vals), size=(csr.n, csr.n)).to("cuda")

    class _Arr:
        def __init__(self, ptr, shape):
            self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f8", "data": (ptr, False),
                                             "version": 3, "strides": None}

    def fn(dev, xp, ldx, yp, ldy, n, m, stream):
        calls.append((dev, m))
        with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=dev)):
            xt = torch.as_tensor(_Arr(xp, (m, ldx)), device=f"cuda:{dev}")[:, :n]
            yt = torch.as_tensor(_Arr(yp, (m, ldy)), device=f"cuda:{dev}")[:, :n]
            yt.copy_(torch.sparse.mm(a, xt.T.contiguous()).T)
        return 0
    return fn


def test_device_callback_config2_family(golden_solves):
    p = P.config2(16)
    calls = []
    K = bosp.LinearOperator.from_device_callback(p.n, _torch_csr_callback(p.K, calls))
    M = bosp.LinearOperator.from_device_callback(p.n, _torch_csr_callback(p.M, calls))
    assert K.kind == bosp.LinearOperator.matrix_free_callback
    res = bosp.solve(K, M, None, bosp.BospConfig(**p.cfg), bosp.GeneralizedNullspace(p.x0, p.y0))
    check_result(res, golden_solves["config2_m16"]["lambdas"], 1e-8, 20)
    assert calls and all(d == 0 for d, _ in calls)
    # block applies of the whole window, not one column at a time
    assert max(m for _, m in calls) >= 20


def test_device_callback_error_status():
    p = P.config2(8)
    good = bosp.LinearOperator.from_csr(p.M)
    bad = bosp.LinearOperator.from_device_callback(p.n, lambda *a: 7)
    with pytest.raises(bosp.BospError, match="device callback returned 7"):
        bosp.solve(bad, good, None, bosp.BospConfig(**p.cfg), bosp.GeneralizedNullspace(p.x0, p.y0))
    # the library stays usable after a failed plugin
    res = bosp.solve(bosp.LinearOperator.from_csr(p.K), good, None, bosp.BospConfig(**p.cfg),
                     bosp.GeneralizedNullspace(p.x0, p.y0))
    assert res.converged


# ---- full-size self-consistency -----------------------------------------------------------

@pytest.mark.slow
def test_config3_full_size_one_vs_two_ranks():
    """Config 3 at 128^3 (n = 2.1 M) as configured: the 1-rank solve and the 2-rank
    row-partitioned solve (halo planes + allreduced Grams, ranks as threads on one GPU) agree,
    and both meet the bar on their own (no reference run exists at this size)."""
    p = P.config3(128, solve=bosp.device_solver)
    cfg = bosp.BospConfig(**p.cfg)
    ns = bosp.GeneralizedNullspace(p.x0, p.y0)
    one = bosp.solve(*bosp.operators_for(p), None, cfg, ns, want_vectors=False)
    two = bosp.solve_multi(2, p.K, p.M, cfg, ns, want_vectors=False)
    for r in (one, two):
        assert r.converged and r.nev_converged == 100
        assert r.residuals.max() < cfg.tol
        assert r.stats["final_biorth_deviation"] < 1e-10
    assert np.abs(one.lambdas - two.lambdas).max() / one.lambdas.max() < 1e-10


# ---- generalized LREP: sparse SPD weight B ---------------------------------

@pytest.mark.parametrize("n", [400, 2000])
def test_weighted_sparse_mass_matrix(n):
    """K x = lambda B y, M y = lambda B x with B the linear-FEM mass matrix (sparse, SPD,
    inner_product.cpp:11-32, kernels.cpp:52-56), the nullspace detected under B -- against the
    unmodified reference's run (tests/golden/golden_weighted_massB_n*.json)."""
    from tests.golden.make_golden_configs import weighted_case
    g = golden(f"weighted_massB_n{n}")
    c = weighted_case(n)
    K = bosp.LinearOperator.from_csr(c["K"])
    M = bosp.LinearOperator.from_csr(c["M"])
    B = bosp.LinearOperator.from_csr(c["B"])
    res = bosp.solve(K, M, bosp.InnerProduct(B), bosp.BospConfig(**c["cfg"]))
    assert res.converged and res.nev_converged == 6
    lam, gl = np.asarray(res.lambdas), np.asarray(g["lambdas"])
    assert np.max(np.abs(lam - gl) / gl) < 1e-10
    assert res.residuals.max() < c["cfg"]["tol"]
    bmat = c["B"].scipy()
    gxy = res.x.T @ (bmat @ res.y)
    assert np.abs(gxy - np.eye(6)).max() < 1e-10
    # the pairs satisfy the generalized equations K x = lambda B y, M y = lambda B x, with the
    # solver's normalisation ||H z - lambda B z|| / ((1 + lambda) ||z||) (bosp_solver.cpp:271)
    r1 = c["K"].scipy() @ res.x - (bmat @ res.y) * lam
    r2 = c["M"].scipy() @ res.y - (bmat @ res.x) * lam
    num = np.sqrt(np.sum(r1 ** 2, 0) + np.sum(r2 ** 2, 0))
    den = (1 + lam) * np.sqrt(np.sum(res.x ** 2, 0) + np.sum(res.y ** 2, 0))
    assert np.max(num / den) < 1e-9
