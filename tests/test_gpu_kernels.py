"""GPU parity of the individual sm_100a kernels against the oracle (numpy restatement of the
reference, pinned by tests/test_oracle.py) and the golden fixtures, through the C ABI."""
import numpy as np
import pytest

from oracle import bosp_oracle as O
from paper_2506_08355_b200 import bosp
from paper_2506_08355_b200 import problems as P
from tests.golden.make_golden import kernel_inputs

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("n,a,b", [(1, 1, 1), (7, 3, 5), (300, 7, 7), (1000, 33, 17),
                                   (4099, 64, 65), (100003, 20, 20), (262144, 60, 60),
                                   (5000, 130, 97)])
def test_gram_matches_numpy(n, a, b):
    rng = np.random.default_rng(n + a + b)
    x = np.asfortranarray(rng.uniform(-1, 1, (n, a)))
    y = np.asfortranarray(rng.uniform(-1, 1, (n, b)))
    g = bosp.block_inner(None, x, y)
    assert rel(g, x.T @ y) < 1e-13


def test_gram_empty_rows():
    g = bosp.block_inner(None, np.zeros((0, 3)), np.zeros((0, 2)))
    assert g.shape == (3, 2) and not g.any()


def test_block_kernels_golden(golden_small):
    x, y = kernel_inputs(1, 300, 7)
    c = np.random.default_rng(2).uniform(-1, 1, (7, 5))
    assert rel(bosp.block_inner(None, x, y), golden_small["inner_xy"]) < 1e-13
    assert rel(bosp.block_product(x, c), golden_small["product_xc"]) < 1e-13
    assert rel(bosp.block_axpy(x, c, y[:, :5]), golden_small["axpy_yxc"]) < 1e-13


@pytest.mark.parametrize("n,k,b", [(5, 2, 1), (1000, 30, 10), (4097, 320, 192), (262144, 60, 20),
                                   (70000, 33, 65)])
def test_product_and_axpy(n, k, b):
    rng = np.random.default_rng(n + k)
    x = np.asfortranarray(rng.uniform(-1, 1, (n, k)))
    c = np.asfortranarray(rng.uniform(-1, 1, (k, b)))
    y = np.asfortranarray(rng.uniform(-1, 1, (n, b)))
    assert rel(bosp.block_product(x, c), x @ c) < 1e-13
    assert rel(bosp.block_axpy(x, c, y), y - x @ c) < 1e-13


def test_dense_operator_apply():
    rng = np.random.default_rng(0)
    for n, m in ((50, 1), (2000, 10), (3001, 33)):
        a = np.asfortranarray(rng.standard_normal((n, n)))
        x = np.asfortranarray(rng.standard_normal((n, m)))
        op = bosp.LinearOperator.from_dense(a)
        assert op.kind == bosp.LinearOperator.dense
        assert rel(op.apply(x), a @ x) < 1e-13


def test_csr_operator_apply_and_spec_examples():
    # T(0) size 3 on ones -> (1,0,1); T(-1) size 4 on ones -> 0
    t0 = bosp.LinearOperator.from_csr(P.t_matrix(3, 0.0))
    assert np.allclose(t0.apply(np.ones(3))[:, 0], [1, 0, 1])
    tm = bosp.LinearOperator.from_csr(P.t_matrix(4, -1.0))
    assert np.abs(tm.apply(np.ones(4))).max() == 0.0
    p = P.config2(16)
    for which in ("K", "M"):
        csr = p.K if which == "K" else p.M
        op = bosp.LinearOperator.from_csr(csr)
        x = np.asfortranarray(np.random.default_rng(1).uniform(-1, 1, (p.n, 9)))
        assert rel(op.apply(x), csr.scipy() @ x) < 1e-14


@pytest.mark.parametrize("grid", [(16, 16, 16), (13, 7, 5), (32, 32, 1), (9, 11, 1)])
@pytest.mark.parametrize("bc,pot", [("neumann", "none"), ("dirichlet", "harmonic"), ("dirichlet", "array")])
def test_stencil_matches_csr(grid, bc, pot):
    nx, ny, nz = grid
    n = nx * ny * nz
    h = 16.0 / (nx + 1)
    v = np.random.default_rng(3).uniform(1, 2, n) if pot == "array" else None
    s = P.Stencil(nx, ny, nz, bc, 1.0 / h ** 2, pot, -8.0, h, v)
    op = bosp.LinearOperator.from_stencil(s)
    x = np.asfortranarray(np.random.default_rng(4).uniform(-1, 1, (n, 6)))
    assert rel(op.apply(x), s.to_csr().scipy() @ x) < 1e-13


@pytest.mark.parametrize("tag,seed,n,m", [("a", 3, 200, 12), ("b", 4, 64, 30)])
def test_mgs_biorth_golden(golden_small, tag, seed, n, m):
    x, y = kernel_inputs(seed, n, m)
    p, q, kept, dropped = bosp.mgs_biorth(x, y)
    assert list(kept) == list(golden_small[f"mgs_{tag}_kept"])
    # the coefficient-space recurrence differs from the reference's column recurrence by
    # rounding only: measured 1.4e-13 / 3.2e-13 of max|P| (cond(X^T Y) = 25 / 233)
    for got, tag2 in ((p, "p"), (q, "q")):
        want = golden_small[f"mgs_{tag}_{tag2}"]
        assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max()
    assert bosp.biorth_residual(p, q) < 1e-10


def test_mgs_biorth_spec_examples():
    p, q, kept, _ = bosp.mgs_biorth(np.array([[1.0], [0.0]]), np.array([[2.0], [0.0]]))
    assert np.allclose(p[:, 0], [1 / np.sqrt(2), 0]) and np.allclose(q[:, 0], [np.sqrt(2), 0])
    e = np.array([[1.0, 1.0], [0.0, 0.0], [0.0, 0.0]])
    _, _, kept, dropped = bosp.mgs_biorth(e, e)
    assert kept == [0] and dropped == [1]
    eye = np.eye(3)[:, :2]
    p, q, kept, _ = bosp.mgs_biorth(eye, eye)
    assert np.allclose(p, eye) and np.allclose(q, eye) and kept == [0, 1]
    # biorth_residual SPEC.md:177-179: P = Q = [e1, e1] -> 1
    assert np.isclose(bosp.biorth_residual(np.array([[1.0, 1], [0, 0]]), np.array([[1.0, 1], [0, 0]])), 1.0)


def test_mgs_biorth_large_matches_oracle_properties():
    rng = np.random.default_rng(11)
    n, m = 100000, 64
    x = np.asfortranarray(rng.uniform(-1, 1, (n, m)))
    y = np.asfortranarray(rng.uniform(-1, 1, (n, m)))
    p, q, kept, dropped = bosp.mgs_biorth(x, y)
    assert len(kept) == m and not dropped
    assert bosp.biorth_residual(p, q) < 1e-10
    # span preservation: x_j in span(P), y_j in span(Q)
    for a, b in ((x, p), (y, q)):
        coef, *_ = np.linalg.lstsq(b, a, rcond=None)
        assert np.abs(b @ coef - a).max() / np.abs(a).max() < 1e-10


def test_cgs_biorth_matches_oracle():
    x, y = kernel_inputs(21, 120, 8)
    p, q, kept, _ = bosp.cgs_biorth(x, y)
    po, qo, ko, _ = O.cgs_biorth(x, y)
    assert kept == ko
    assert np.allclose(p, po, rtol=1e-8, atol=1e-9)


def test_biorth_against_golden(golden_small):
    x, y = kernel_inputs(5, 150, 6)
    bx, by = kernel_inputs(6, 150, 4)
    cx, cy = kernel_inputs(7, 150, 3)
    bp, bq, _, _ = O.mgs_biorth(bx, by)
    cp, cq, _, _ = O.mgs_biorth(cx, cy)
    w, z = bosp.biorth_against([(bp, bq), (cp, cq)], x, y)
    assert np.allclose(w, golden_small["against_w"], rtol=1e-10, atol=1e-11)
    assert np.allclose(z, golden_small["against_z"], rtol=1e-10, atol=1e-11)
    # basis (e1, e1), X = Y = e1 -> 0
    e1 = np.array([[1.0], [0.0], [0.0]])
    w, z = bosp.biorth_against([(e1, e1)], e1, e1)
    assert not w.any() and not z.any()


def test_cg_golden_and_masks(golden_small):
    t = bosp.LinearOperator.from_csr(P.t_matrix(50, 0.0))
    rhs = np.random.default_rng(8).uniform(-1, 1, (50, 4))
    for tol, it in ((1e-2, 20), (1e-12, 100)):
        x, br, mi = bosp.cg_solve(t, rhs, tol=tol, max_iter=it)
        assert mi == int(golden_small[f"cg_{it}_maxit"][0])
        assert np.allclose(x, golden_small[f"cg_{it}"], rtol=1e-9, atol=1e-10)
    # rhs = 0 -> 0; 2I -> b/2 in one iteration
    x, br, mi = bosp.cg_solve(t, np.zeros((50, 2)))
    assert not x.any() and mi == 0
    two = bosp.LinearOperator.scaled_identity(5, 2.0)
    b = np.arange(1.0, 6.0)[:, None]
    x, br, mi = bosp.cg_solve(two, b, tol=1e-12, max_iter=10)
    assert np.allclose(x, b / 2) and mi == 1
    # mixed columns: one zero rhs column stays exactly zero
    rhs2 = np.concatenate([rhs[:, :2], np.zeros((50, 1)), rhs[:, 2:]], axis=1)
    x2, _, _ = bosp.cg_solve(t, rhs2, tol=1e-2, max_iter=20)
    assert not x2[:, 2].any()
    assert np.allclose(x2[:, [0, 1, 3, 4]], golden_small["cg_20"], rtol=1e-9, atol=1e-10)


def test_cg_breakdown_on_spsd():
    # K = T(-1) is singular along ones: CG on rhs = ones hits p^T A p = 0 -> breakdown, x stays 0
    k = bosp.LinearOperator.from_csr(P.t_matrix(8, -1.0))
    x, br, mi = bosp.cg_solve(k, np.ones((8, 1)), tol=1e-12, max_iter=10)
    xo, bo, mo = O.cg_solve(O.op_from_spec(P.t_matrix(8, -1.0).spec()), np.ones((8, 1)),
                            np.zeros((8, 1)), 1e-12, 10)
    assert br == bo and mi == mo
    assert np.allclose(x, xo)


def test_small_lrep_host(golden_small):
    lam, xh, yh = bosp.solve_small_lrep(golden_small["small_k"], golden_small["small_m"], 5)
    assert np.allclose(lam, golden_small["small_lam"], rtol=1e-13)
    assert np.allclose(xh.T @ yh, np.eye(5), atol=1e-12)
    lam, xh, yh = bosp.solve_small_lrep(np.array([[4.0]]), np.array([[9.0]]), 1)
    assert np.isclose(lam[0], 6.0) and np.isclose(yh[0, 0], 2 / np.sqrt(6))
    with pytest.raises(bosp.NullspaceLeak):
        bosp.solve_small_lrep(np.array([[-1.0]]), np.array([[1.0]]), 1)


def test_weighted_inner_product():
    rng = np.random.default_rng(5)
    n = 200
    d = rng.uniform(1, 2, n)
    B = bosp.LinearOperator.diagonal(d)
    ip = bosp.InnerProduct(B)
    x = rng.uniform(-1, 1, (n, 4))
    y = rng.uniform(-1, 1, (n, 3))
    assert rel(bosp.block_inner(ip, x, y), x.T @ (d[:, None] * y)) < 1e-13
    p, q, kept, _ = bosp.mgs_biorth(x[:, :3], y, ip)
    assert np.abs(p.T @ (d[:, None] * q) - np.eye(3)).max() < 1e-12


def test_seed_blocks_bit_exact_reference_stream(golden_small):
    """Device MT19937-64 fill == the reference's fill_uniform stream (x,p,w,y,q,z order)."""
    n, d = 100, 10  # 2 * 100 * 10 = 2000 draws = golden rng_seed0
    u, v = bosp.seed_blocks(0, n, d)
    stream = np.concatenate([u.T.reshape(-1), v.T.reshape(-1)])
    assert np.array_equal(stream, golden_small["rng_seed0"])
    # longer stream against the oracle restatement (crosses many 312-word twists)
    u, v = bosp.seed_blocks(12345, 4099, 3)
    ref = O.MT19937_64(12345).uniform(2 * 4099 * 3)
    assert np.array_equal(np.concatenate([u.T.reshape(-1), v.T.reshape(-1)]), ref)


def test_seed_blocks_jump_ahead_long_stream():
    """17.3M draws: ~130 CTAs each jump to their 2^16-draw segments with both polynomial tables
    (segment index >= 256 uses table B then A) -- still the reference's single stream."""
    n, d = 262147, 33
    u, v = bosp.seed_blocks(7, n, d)
    got = np.concatenate([u.T.reshape(-1), v.T.reshape(-1)])
    ref = O.MT19937_64(7).uniform(2 * n * d)
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, (bad.size, bad[:5])


def test_shape_errors_map_to_contract_violation():
    with pytest.raises(bosp.ContractViolation):
        bosp.block_inner(None, np.ones((5, 2)), np.ones((4, 2)))
    with pytest.raises(bosp.ContractViolation):
        bosp.block_product(np.ones((5, 2)), np.ones((3, 2)))
    op = bosp.LinearOperator.identity(4)
    with pytest.raises(bosp.ContractViolation):
        op.apply(np.ones((5, 1)))


@pytest.mark.parametrize("case", ["stencil_csr", "banded_varying", "holes", "sym_holes", "tridiag_holes", "sym_const", "wide_band"])
def test_csr_storage_formats_apply(case):
    """Banded CSR goes to DIA (constant diagonals + presence mask), everything else to SELL-32;
    both must reproduce the CSR products (scipy) to rounding."""
    import scipy.sparse as sp
    rng = np.random.default_rng(5)
    if case == "stencil_csr":
        a = P.config2(16).M.scipy()
    elif case == "banded_varying":
        n = 5000
        offs = [-70, -3, -1, 0, 1, 2, 70]
        a = sp.diags([rng.standard_normal(n - abs(o)) for o in offs], offs, shape=(n, n), format="csr")
    elif case == "holes":
        n = 4000
        offs = [-9, -1, 0, 1, 9]
        a = sp.diags([rng.standard_normal(n - abs(o)) for o in offs], offs, shape=(n, n), format="lil")
        for i in rng.integers(0, n - 10, 300):
            a[i, i + 1] = 0.0
        a = a.tocsr()
        a.eliminate_zeros()
    elif case in ("sym_holes", "tridiag_holes", "sym_const"):
        # the banded pair kernel's layout: offsets (.., -1, 0, 1, ..) with the others even;
        # sym_const: every diagonal constant (coefficients from the constant bank)
        n = 4096
        offs = [-1, 0, 1] if case == "tridiag_holes" else [-512, -10, -1, 0, 1, 10, 512]
        vals = ([np.full(n - abs(o), 0.5 + k) for k, o in enumerate(offs)] if case == "sym_const"
                else [rng.standard_normal(n - abs(o)) for o in offs])
        a = sp.diags(vals, offs, shape=(n, n), format="lil")
        for i in rng.integers(0, n - 12, 300):
            a[i, i + 1] = 0.0
            a[i + 11, i + 1] = 0.0
        a = a.tocsr()
        a.eliminate_zeros()
    else:  # 20 diagonals -> more than the DIA limit -> SELL
        n = 3000
        offs = list(range(-10, 10))
        a = sp.diags([rng.standard_normal(n - abs(o)) + 1.0 for o in offs], offs, shape=(n, n), format="csr")
    a.sort_indices()
    op = bosp.LinearOperator.from_csr(a.indptr.astype(np.int64), a.indices.astype(np.int64), a.data)
    x = np.asfortranarray(rng.standard_normal((a.shape[0], 7)))
    y = op.apply(x)
    ref = a @ x
    assert np.abs(y - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())


GRAM_WIDTHS = [1, 8, 9, 17, 24, 25, 32, 33, 40, 41, 48, 49, 56, 57, 64, 65]


@pytest.mark.parametrize("a", GRAM_WIDTHS)
def test_gram_width_sweep(a):
    """Every Gram dispatch class (single-warp-group register tiles, 2x1 / 1x2 / 2x2 warp
    groups, the shared-memory tiled kernel) against numpy, with odd row counts."""
    rng = np.random.default_rng(a)
    n = 3001 + 7 * a
    x = np.asfortranarray(rng.uniform(-1, 1, (n, a)))
    for b in GRAM_WIDTHS:
        y = np.asfortranarray(rng.uniform(-1, 1, (n, b)))
        assert rel(bosp.block_inner(None, x, y), x.T @ y) < 1e-13, (a, b)


@pytest.mark.parametrize("k", [1, 7, 8, 20, 33, 60, 64, 65, 100])
def test_product_width_sweep(k):
    rng = np.random.default_rng(100 + k)
    n = 5003
    x = np.asfortranarray(rng.uniform(-1, 1, (n, k)))
    for b in (1, 8, 9, 20, 24, 33, 48, 60, 64, 65):
        c = np.asfortranarray(rng.uniform(-1, 1, (k, b)))
        y = np.asfortranarray(rng.uniform(-1, 1, (n, b)))
        assert rel(bosp.block_product(x, c), x @ c) < 1e-13, (k, b)
        assert rel(bosp.block_axpy(x, c, y), y - x @ c) < 1e-13, (k, b)


@pytest.mark.parametrize("a,b", [(20, 20), (33, 33), (40, 40), (48, 48), (40, 8), (60, 60), (64, 64), (64, 20), (96, 64)])
@pytest.mark.parametrize("nseg", [1, 3])
def test_gram_multi_job_segments(a, b, nseg):
    """The MGS / drift-monitor Gram triple in one launch, X in column segments."""
    rng = np.random.default_rng(a * 100 + b + nseg)
    n = 20011
    x = np.asfortranarray(rng.uniform(-1, 1, (n, a)))
    y = np.asfortranarray(rng.uniform(-1, 1, (n, b)))
    for njobs in (1, 2, 3):
        g1, g2, g3 = bosp._test_gram_jobs(x, y, nseg, njobs)
        assert rel(g1, x.T @ y) < 1e-13, (njobs, "xy")
        if njobs > 1:
            assert rel(g2, x.T @ x) < 1e-13, (njobs, "xx")
        if njobs > 2:
            assert rel(g3, y.T @ y) < 1e-13, (njobs, "yy")


@pytest.mark.parametrize("full", [False, True])
@pytest.mark.parametrize("k,kb", [(1, 1), (4, 4), (7, 5), (8, 8), (12, 9), (12, 12), (16, 16), (20, 20), (24, 17),
                                  (24, 24), (32, 32), (20, 2)])
@pytest.mark.parametrize("n", [1, 63, 5003, 8192, 8321, 262147])
def test_biorth_apply_fused(k, kb, n, full):
    """MGS-Biorth application fused with its check Gram: P = X A, Q = Y B, P^T Q in one kernel
    (biorth.cpp:19-69 / :104-107) against numpy; row counts with a partial last 64- / 128-row
    tile, upper-triangular coefficients (the kernels' triangular K loops) and full ones, every
    compile-time width pair of k_biorth_apply4 plus the runtime-width and TMA kernels."""
    rng = np.random.default_rng(7 * k + kb + n)
    x = np.asfortranarray(rng.uniform(-1, 1, (n, k)))
    y = np.asfortranarray(rng.uniform(-1, 1, (n, k)))
    a = np.asfortranarray(rng.uniform(-1, 1, (k, kb)))
    b = np.asfortranarray(rng.uniform(-1, 1, (k, kb)))
    if not full:
        a, b = np.asfortranarray(np.triu(a)), np.asfortranarray(np.triu(b))
    p, q, g = bosp._test_biorth_apply(x, y, a, b)
    pr, qr = x @ a, y @ b
    assert rel(p, pr) < 1e-13 and rel(q, qr) < 1e-13
    assert rel(g, pr.T @ qr) < 1e-12


@pytest.mark.parametrize("a", [1, 4, 10, 16, 20, 24, 28, 30, 60, 160])
@pytest.mark.parametrize("n", [7, 20011, 262147])
def test_gram_symmetric(a, n):
    """Symmetric Grams (upper tiles mirrored): the MGS pair Gram of Z = [X | Y] (register path up
    to 48 columns of Z, tiled beyond) and a U^T (K U)-style Gram with distinct operands."""
    rng = np.random.default_rng(31 * a + n)
    x = np.asfortranarray(rng.uniform(-1, 1, (n, a)))
    y = np.asfortranarray(rng.uniform(-1, 1, (n, a)))
    z = np.hstack([x, y])
    g = bosp._test_gram_sym(x, y, same=True)
    assert np.array_equal(g, g.T)
    assert rel(g, z.T @ z) < 1e-13
    d = rng.uniform(0.5, 2.0, n)
    ky = np.asfortranarray(d[:, None] * x)        # K = diag(d): X^T (K X) is symmetric
    h = bosp._test_gram_sym(x, ky, same=False)
    ref = x.T @ ky
    assert np.array_equal(h, h.T)
    assert rel(h, 0.5 * (ref + ref.T)) < 1e-13


@pytest.mark.parametrize("m", [2, 8, 20, 32])
@pytest.mark.parametrize("n", [8192, 100003])
def test_mgs_device_coefficients(m, n):
    """The solver's MGS-Biorth for m <= 32 (pair Gram on bulk-async staging -> LDU coefficients
    on the device -> fused application): same kept set as the oracle's gs_biorth
    (biorth.cpp:19-69), P, Q equal to it up to the recurrence's rounding, biorthogonal."""
    rng = np.random.default_rng(m * 1000 + n % 997)
    x = np.asfortranarray(rng.uniform(-1, 1, (n, m)))
    y = np.asfortranarray(x + 0.5 * rng.uniform(-1, 1, (n, m)))
    p, q, second = bosp._test_mgs_dev(x, y)
    po, qo, ko, do = O.mgs_biorth(x, y)
    assert p.shape[1] == len(ko) == m and not do
    assert rel(p, po) < 1e-10 and rel(q, qo) < 1e-10
    assert np.abs(p.T @ q - np.eye(m)).max() < 1e-12


def test_mgs_device_coefficients_fallback():
    """A nearly dependent column (cancellation) and an exact duplicate (drop) are decided by the
    host's column-sequential recurrence, as gs_biorth does in n-space: same kept/dropped sets."""
    rng = np.random.default_rng(5)
    n, m = 20000, 12
    x = np.asfortranarray(rng.uniform(-1, 1, (n, m)))
    x[:, 7] = x[:, 3]                              # exact duplicate -> dropped
    x[:, 9] = x[:, 1] + 1e-9 * rng.uniform(-1, 1, n)  # cancels in coefficient space
    y = np.asfortranarray(x + 0.25 * rng.uniform(-1, 1, (n, m)))
    y[:, 7] = y[:, 3]
    p, q, _ = bosp._test_mgs_dev(x, y)
    po, qo, ko, do = O.mgs_biorth(x, y)
    assert p.shape[1] == len(ko)
    assert np.abs(p.T @ q - np.eye(len(ko))).max() < 1e-10


@pytest.mark.parametrize("k", [1, 3, 8])
@pytest.mark.parametrize("b", [65, 320])
@pytest.mark.parametrize("n", [7, 20011])
def test_rank_k_product_and_axpy(k, b, n):
    """Rank-k updates of wide blocks (the streaming k <= 8 path: the projection of a d-column
    block against the null basis) against numpy: block_product (kernels.cpp:70-87) and
    block_axpy (:89-104), odd n included."""
    rng = np.random.default_rng(100 * k + b + n)
    x = np.asfortranarray(rng.uniform(-1, 1, (n, k)))
    c = np.asfortranarray(rng.uniform(-1, 1, (k, b)))
    y = np.asfortranarray(rng.uniform(-1, 1, (n, b)))
    assert rel(bosp.block_product(x, c), x @ c) < 1e-14
    assert rel(bosp.block_axpy(x, c, y), y - x @ c) < 1e-14

