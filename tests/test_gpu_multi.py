"""Row-partitioned solves against the unpartitioned solve and the reference.

Every n-length block is split by rows over `nranks` ranks; Grams/dots are allreduced, sparse
applies exchange halo rows, dense applies allgather X.  Here the ranks are threads of one
process sharing the single B200 of the test box (ThreadComm over device memory), which runs
exactly the partitioned code path a multi-GPU NCCL run takes, minus the transport.  The bar is
the solver's: eigenvalues within 1e-10 relative of the reference, residuals below tol,
max |X^T Y - I| below 1e-10 -- and agreement with the one-rank solve.
"""
import numpy as np
import pytest

from paper_2506_08355_b200 import bosp
from paper_2506_08355_b200 import problems as P
from tests.test_gpu_solver import check_result

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_partitioned_csr_config2(golden_solves, nranks):
    p = P.config2(16)
    cfg = bosp.BospConfig(**p.cfg)
    res = bosp.solve_multi(nranks, p.K, p.M, cfg, bosp.GeneralizedNullspace(p.x0, p.y0))
    check_result(res, golden_solves["config2_m16"]["lambdas"], 1e-8, 20)


@pytest.mark.parametrize("nranks", [2, 4])
def test_partitioned_stencil3d_matches_serial(golden_solves, nranks):
    p = P.config2(16)
    kop, mop = P._grid3_ops(16)
    cfg = bosp.BospConfig(**p.cfg)
    ns = bosp.GeneralizedNullspace(p.x0, p.y0)
    serial = bosp.solve(bosp.LinearOperator.from_stencil(kop), bosp.LinearOperator.from_stencil(mop), None,
                        cfg, ns)
    res = bosp.solve_multi(nranks, kop, mop, cfg, ns)
    check_result(res, golden_solves["config2_m16"]["lambdas"], 1e-8, 20)
    assert np.abs(res.lambdas - serial.lambdas).max() / serial.lambdas.max() < 1e-11
    # same random start; allreduce summation order perturbs roundoff, so the trajectories
    # (drops, repairs) may drift apart a little, not the converged eigenvalues
    assert res.iterations <= 1.5 * serial.iterations


def test_partitioned_stencil2d_moving(golden_solves):
    """Config-5 family (5-point, array potential) with moving/locking over 2 ranks."""
    p = P.config5(32)
    cfg = bosp.BospConfig(nev=40, nb=8, tol=1e-8)
    assert cfg.effective_moving()
    res = bosp.solve_multi(2, p.K, p.M, cfg, bosp.GeneralizedNullspace(p.x0, p.y0))
    check_result(res, golden_solves["config5_m32"]["lambdas"], 1e-8, 40)


def test_partitioned_dense_config1(golden_solves):
    p = P.config1()
    res = bosp.solve_multi(2, p.K, p.M, bosp.BospConfig(**p.cfg), bosp.GeneralizedNullspace(p.x0, p.y0))
    check_result(res, golden_solves["config1"]["lambdas"], 1e-8, 10)


def test_partitioned_table3(golden_solves):
    n = 1000
    res = bosp.solve_multi(3, P.t_matrix(n, -1.0), P.t_matrix(n, 0.0), bosp.BospConfig(nev=10, nb=10, tol=1e-10),
                           bosp.GeneralizedNullspace(*P.analytic_nullspace_T(n)))
    check_result(res, golden_solves["tm1_t0_n1000"]["lambdas"], 1e-10, 10)


def test_partitioned_computes_nullspace():
    """No nullspace given: every rank runs the partitioned compute_nullspace first."""
    n = 200
    t = P.t_matrix(n, 0.0)
    res = bosp.solve_multi(2, t, t, bosp.BospConfig(nev=4, nb=4, tol=1e-10))
    assert res.converged
    assert np.allclose(res.lambdas, P.t_eigenvalues(n, 4), rtol=1e-11)


def test_partitioned_ragged_rows(golden_solves):
    """n = 401 over 4 ranks: slices of 100, 100, 100, 101 rows."""
    n = 401
    k, m = P.t_matrix(n, -1.0), P.t_matrix(n, 0.0)
    ns = bosp.GeneralizedNullspace(*P.analytic_nullspace_T(n))
    cfg = bosp.BospConfig(nev=5, nb=5, tol=1e-10)
    serial = bosp.solve(bosp.LinearOperator.from_csr(k), bosp.LinearOperator.from_csr(m), None, cfg, ns)
    res = bosp.solve_multi(4, k, m, cfg, ns)
    check_result(res, golden_solves["tm1_t0_n401"]["lambdas"], 1e-10, 5)
    assert np.allclose(res.lambdas, serial.lambdas, rtol=1e-12)


def test_partitioned_errors():
    t = P.t_matrix(50, 0.0)
    with pytest.raises(bosp.ContractViolation):
        bosp.solve_multi(17, t, t, bosp.BospConfig(nev=2, nb=2))
    with pytest.raises(bosp.ContractViolation):
        bosp.solve_multi(2, t, P.t_matrix(60, 0.0), bosp.BospConfig(nev=2, nb=2))


def test_nccl_single_rank_comm(golden_solves):
    """NCCL bootstrap on one GPU: unique id, a 1-rank communicator attached to this thread,
    then a solve through it (the multi-GPU bench path with N = 1)."""
    uid = bosp.comm_nccl_unique_id()
    assert len(uid) == 128
    n = 300
    k, m = P.t_matrix(n, -1.0), P.t_matrix(n, 0.0)
    bosp.comm_init_nccl(uid, 1, 0, n, 0)
    try:
        res = bosp.solve(bosp.local_operator(k, 1, 0), bosp.local_operator(m, 1, 0), None,
                         bosp.BospConfig(nev=4, nb=4, tol=1e-10), bosp.GeneralizedNullspace(*P.analytic_nullspace_T(n)))
    finally:
        bosp.comm_free()
    check_result(res, golden_solves["tm1_t0_n300"]["lambdas"], 1e-10, 4)


# ---- the round-2 config families under the row partition ----------------------------------

def test_partitioned_config5_as_configured():
    """Config 5 as configured (nev 500, nb 64, moving with repeated locking, d = 320) at 64^2 over
    2 ranks (grid rows split, halo rows, allreduced Grams, grouped locked-basis projections)
    against the unmodified reference's run (tests/golden/golden_config5_m64.json)."""
    from tests.test_gpu_configs import golden
    g = golden("config5_m64")
    p = P.config5(64)
    res = bosp.solve_multi(2, p.K, p.M, bosp.BospConfig(**p.cfg), bosp.GeneralizedNullspace(p.x0, p.y0))
    check_result(res, g["lambdas"], 1e-8, 500)


def test_partitioned_config4_dense():
    """Config 4's dense BSE-like family at n = 4096 over 2 ranks (allgather of X, each rank's rows
    of A^T) against the reference (tests/golden/golden_config4_n4096.json)."""
    from tests.test_gpu_configs import golden
    g = golden("config4_n4096")
    p = P.config4(n=4096)
    res = bosp.solve_multi(2, p.K, p.M, bosp.BospConfig(**p.cfg), bosp.GeneralizedNullspace(p.x0, p.y0))
    check_result(res, g["lambdas"], 1e-8, 32)


def test_partitioned_config3_as_configured_m32():
    from tests.test_gpu_configs import golden
    g = golden("config3_m32")
    p = P.config3(32)
    res = bosp.solve_multi(4, p.K, p.M, bosp.BospConfig(**p.cfg), bosp.GeneralizedNullspace(p.x0, p.y0))
    check_result(res, g["lambdas"], 1e-8, 100)


@pytest.mark.parametrize("nranks", [2, 3])
def test_partitioned_weighted_sparse_B(nranks):
    """SURVEY 8(f)2 under the row partition: the sparse FEM mass matrix B applied per rank (halo
    rows like K and M), nullspace detected by the partitioned detector under B, against the
    unmodified reference's run (tests/golden/golden_weighted_massB_n2000.json)."""
    from tests.golden.make_golden_configs import weighted_case
    from tests.test_gpu_configs import golden
    g = golden("weighted_massB_n2000")
    c = weighted_case(2000)
    res = bosp.solve_multi(nranks, c["K"], c["M"], bosp.BospConfig(**c["cfg"]), B=c["B"])
    assert res.converged and res.nev_converged == 6
    assert np.max(np.abs(res.lambdas - np.asarray(g["lambdas"])) / np.asarray(g["lambdas"])) < 1e-10
    assert res.residuals.max() < c["cfg"]["tol"]
    gxy = res.x.T @ (c["B"].scipy() @ res.y)
    assert np.abs(gxy - np.eye(6)).max() < 1e-10


_HALO_SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r})
from paper_2506_08355_b200 import bosp, problems as P
p = P.config2(16)
kop, mop = P._grid3_ops(16)
res = bosp.solve_multi(3, kop, mop, bosp.BospConfig(**p.cfg), bosp.GeneralizedNullspace(p.x0, p.y0))
print(json.dumps({{"lambdas": list(map(float, res.lambdas)), "iterations": int(res.iterations),
                  "converged": bool(res.converged)}}))
"""


def test_stencil_halo_overlap_matches_exchange_first():
    """Slab-partitioned stencil apply with the halo exchange overlapped with the interior planes
    (interior launch, exchange on a side stream, boundary-plane launches sharing the dot
    partials) against the exchange-first single launch (BOSP_HALO_OVERLAP=0): the
    split changes no row's arithmetic, only the order of the p^T A p partials, so the solves
    agree to rounding.  3 ranks: a middle slab with both halos.  (The switch is read once per
    process, hence the subprocesses.)"""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("1", "0"):
        env = dict(os.environ, BOSP_HALO_OVERLAP=mode)
        r = subprocess.run([sys.executable, "-c", _HALO_SCRIPT.format(root=root)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[mode] = json.loads(r.stdout.strip().splitlines()[-1])
    a, b = np.array(out["1"]["lambdas"]), np.array(out["0"]["lambdas"])
    assert out["1"]["converged"] and out["0"]["converged"]
    assert np.abs(a - b).max() / np.abs(b).max() < 1e-11
