"""Seeded generators for the five BASELINE.json configurations (and the paper's T(s) family).

Nothing here is on the solver's hot path: these build K, M and the explicit generalized
nullspace (X0, Y0) that BOTH the B200 solver and the CPU oracle receive, so the two sides
always see bit-identical inputs.  Conventions (written down once):

* T(s)          -- PAPER.md:1681-1693: tridiag(-1, 2, -1) with corner entries s.
* config 1      -- dense n=2000: K = Q diag(dK) Q^T (Q from QR of N(0,1)), dK = 10 zeros +
                   1990 U[0.1, 10]; M = G G^T / n + I.  Lower triangles mirrored -> exactly
                   symmetric.  X0 = Q[:, zero indices].
* configs 2/3   -- m^3 grid, nodes x_i = -8 + i*h (i = 1..m), h = 16/(m+1), lexicographic
                   index i + m*(j + m*k).  K = Neumann graph Laplacian / h^2 (diag = number of
                   in-grid neighbours, off-diagonal -1), M = Dirichlet 7-point Laplacian / h^2 +
                   diag(0.5 |x|^2).  N(K) = constants.
* config 4      -- dense BSE-like n=16384: A = diag(eps) + V V^T, B = W W^T; N = random
                   orthonormal n x 64, Pi = I - N N^T, K = Pi (A - B) Pi, M = A + B.  X0 = N.
* config 5      -- 1024^2 5-point grid, h = 1: K = Neumann graph Laplacian, M = Dirichlet
                   Laplacian + diag(1 + u), u ~ U[0, 1].  N(K) = constants.

The nullspace pair is normalised exactly as the reference's compute_nullspace does
(nullspace.cpp:173-190): Y = M^-1 X, G = sym(X^T Y), C = chol(G)^T, X0 = X C^-1, Y0 = Y C^-1.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

DEFAULT_SEED = 2025


@dataclass
class Csr:
    """CSR with int64 row offsets / column indices (sorted, strictly increasing per row)."""
    n: int
    rowptr: np.ndarray
    colidx: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    def spec(self):
        return ("csr", (self.rowptr, self.colidx, self.vals))

    def scipy(self):
        return sp.csr_matrix((self.vals, self.colidx, self.rowptr), shape=(self.n, self.n))


def csr_from_scipy(a) -> Csr:
    a = sp.csr_matrix(a)
    a.sum_duplicates()
    a.sort_indices()
    return Csr(a.shape[0], a.indptr.astype(np.int64), a.indices.astype(np.int64),
               a.data.astype(np.float64))


@dataclass
class Stencil:
    """Matrix-free Laplacian-family operator on a structured grid (applied by the B200 stencil
    kernel; its CSR twin feeds the oracle).

    y = scale * (L_bc x) + diag(v) x, where L_bc is the Neumann graph Laplacian ("neumann") or
    the Dirichlet Laplacian ("dirichlet") on an nx*ny*nz grid (nz = 1 -> 5-point), and v is
    either 0, the harmonic potential 0.5*|x|^2 of the node coordinates (computed on the fly),
    or an explicit per-node array.
    """
    nx: int
    ny: int
    nz: int
    bc: str                      # "neumann" | "dirichlet"
    scale: float                 # 1/h^2
    potential: str = "none"      # "none" | "harmonic" | "array"
    origin: float = 0.0          # coordinate of node index -1 (x_i = origin + (i+1)*h)
    h: float = 1.0
    v: np.ndarray | None = None  # explicit diagonal (potential == "array")

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.nz

    def diag_potential(self) -> np.ndarray:
        if self.potential == "none":
            return np.zeros(self.n)
        if self.potential == "array":
            return np.asarray(self.v, dtype=np.float64)
        c = [self.origin + (np.arange(m) + 1) * self.h for m in (self.nx, self.ny, self.nz)]
        x = c[0][None, None, :]
        y = c[1][None, :, None]
        z = c[2][:, None, None] if self.nz > 1 else np.zeros((1, 1, 1))
        return (0.5 * (x * x + y * y + z * z)).reshape(-1) * np.ones(self.n)

    def to_csr(self) -> Csr:
        dims = [self.nx, self.ny] + ([self.nz] if self.nz > 1 else [])
        a = _grid_laplacian(dims, self.bc) * self.scale
        a = a + sp.diags(self.diag_potential())
        return csr_from_scipy(a)


def _grid_laplacian(dims, bc):
    """Graph (neumann) or Dirichlet Laplacian on a tensor grid, index = i + nx*(j + ny*k)."""
    ops = []
    for m in dims:
        e = np.ones(m)
        path = sp.diags([-e[:-1], -e[:-1]], [-1, 1], shape=(m, m))
        deg = np.full(m, 2.0)
        if bc == "neumann":
            deg[0] = deg[-1] = 1.0
        ops.append((path, deg))
    n = int(np.prod(dims))
    a = sp.csr_matrix((n, n))
    for ax, (path, deg) in enumerate(ops):
        term = None
        for bx, (p2, d2) in enumerate(ops):
            f = (path + sp.diags(deg)) if ax == bx else sp.identity(dims[bx])
            # kron order: last axis (slowest) first
            term = f if term is None else sp.kron(f, term)
        a = a + term
    return a.tocsr()


def t_matrix(n: int, s: float) -> Csr:
    """T(s)."""
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i); cols.append(i); vals.append(2.0)
        if i > 0:
            rows.append(i); cols.append(i - 1); vals.append(-1.0)
        if i + 1 < n:
            rows.append(i); cols.append(i + 1); vals.append(-1.0)
    if s != 0.0 and n > 2:
        rows += [0, n - 1]; cols += [n - 1, 0]; vals += [s, s]
    a = sp.coo_matrix((vals, (rows, cols)), shape=(n, n))
    return csr_from_scipy(a)


def t_eigenvalues(n: int, count: int) -> np.ndarray:
    """Exact lambda_l = 4 sin^2(pi l / (2(n+1))) for K = M = T(0)."""
    l = np.arange(1, count + 1)
    return 4.0 * np.sin(np.pi * l / (2.0 * (n + 1))) ** 2


def analytic_nullspace_T(n: int):
    """x0 = ones, y0_l = l(n-l+1)/2, scaled so x0^T y0 = 1 (nullspace.cpp:195-212)."""
    l = np.arange(1, n + 1, dtype=np.float64)
    a = l * (n - l + 1) / 2.0
    s = 1.0 / np.sqrt(a.sum())
    return (np.ones((n, 1)) * s).copy(order="F"), (a[:, None] * s).copy(order="F")


def normalize_nullspace(x_raw: np.ndarray, y_raw: np.ndarray):
    """G = sym(X^T Y) = C^T C, X0 = X C^-1, Y0 = Y C^-1 (nullspace.cpp:179-190)."""
    g = x_raw.T @ y_raw
    g = 0.5 * (g + g.T)
    l = np.linalg.cholesky(g)
    cinv = np.linalg.inv(l.T)
    return np.asfortranarray(x_raw @ cinv), np.asfortranarray(y_raw @ cinv)


def _cg_solve_sparse(m, b, rtol=1e-13):
    out = np.zeros_like(b)
    for j in range(b.shape[1]):
        x, info = spla.cg(m, b[:, j], rtol=rtol, atol=0.0, maxiter=20 * m.shape[0])
        if info != 0:
            raise RuntimeError(f"nullspace CG did not converge (info={info})")
        out[:, j] = x
    return out


@dataclass
class Problem:
    name: str
    n: int
    K: object                    # Csr | Stencil | np.ndarray (dense, column-major)
    M: object
    x0: np.ndarray
    y0: np.ndarray
    cfg: dict
    meta: dict = field(default_factory=dict)

    def oracle_spec(self, which: str):
        """Operator spec for oracle/ref.py (stencils are handed over in CSR form)."""
        op = self.K if which == "K" else self.M
        if isinstance(op, np.ndarray):
            return ("dense", op)
        if isinstance(op, Stencil):
            op = op.to_csr()
        return op.spec()


def config1(seed: int = DEFAULT_SEED, n: int = 2000, nzero: int = 10) -> Problem:
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    dk = np.concatenate([np.zeros(nzero), rng.uniform(0.1, 10.0, n - nzero)])
    k = (q * dk) @ q.T
    g = rng.standard_normal((n, n))
    m = g @ g.T / n + np.eye(n)
    for a in (k, m):
        il = np.tril_indices(n, -1)
        a.T[il] = a[il]          # mirror lower onto upper: exactly symmetric
    k = np.asfortranarray(k)
    m = np.asfortranarray(m)
    x_raw = np.asfortranarray(q[:, :nzero])
    y_raw = np.linalg.solve(m, x_raw)
    x0, y0 = normalize_nullspace(x_raw, y_raw)
    cfg = dict(nev=10, nb=20, tol=1e-8)
    return Problem("config1-dense-n2000", n, k, m, x0, y0, cfg, dict(seed=seed))


def _grid3_ops(m: int):
    h = 16.0 / (m + 1)
    kop = Stencil(m, m, m, "neumann", 1.0 / h ** 2, "none", -8.0, h)
    mop = Stencil(m, m, m, "dirichlet", 1.0 / h ** 2, "harmonic", -8.0, h)
    return kop, mop


def _constant_nullspace(mop, n: int, solve=None):
    """X0 ∝ constants (N of the Neumann graph Laplacian); Y0 = M^-1 X0 by `solve(M)` (a factory
    M -> (b -> M^-1 b), e.g. bosp.device_solver on a GPU box) or scipy CG on the CSR form."""
    x_raw = np.full((n, 1), 1.0 / np.sqrt(n))
    if solve is not None:
        y_raw = solve(mop)(x_raw)
    else:
        mcsr = mop.to_csr() if isinstance(mop, Stencil) else mop
        y_raw = _cg_solve_sparse(mcsr.scipy(), x_raw)
    return normalize_nullspace(x_raw, y_raw)


def config2(m: int = 64, solve=None) -> Problem:
    kop, mop = _grid3_ops(m)
    kc, mc = kop.to_csr(), mop.to_csr()
    x0, y0 = _constant_nullspace(mc, kc.n, solve)
    cfg = dict(nev=20, nb=40, tol=1e-8)
    return Problem(f"config2-csr-{m}^3", kc.n, kc, mc, x0, y0, cfg, dict(grid=m))


def config3(m: int = 128, solve=None, nev: int = 100) -> Problem:
    kop, mop = _grid3_ops(m)
    x0, y0 = _constant_nullspace(mop, kop.n, solve)
    cfg = dict(nev=nev, nb=64, tol=1e-8, moving=True)
    return Problem(f"config3-stencil7-{m}^3", kop.n, kop, mop, x0, y0, cfg, dict(grid=m))


def config5(m: int = 1024, seed: int = DEFAULT_SEED, solve=None, nev: int = 500) -> Problem:
    rng = np.random.default_rng(seed)
    u = rng.uniform(0.0, 1.0, m * m)
    kop = Stencil(m, m, 1, "neumann", 1.0)
    mop = Stencil(m, m, 1, "dirichlet", 1.0, "array", v=1.0 + u)
    x0, y0 = _constant_nullspace(mop, kop.n, solve)
    cfg = dict(nev=nev, nb=64, tol=1e-8)
    return Problem(f"config5-stencil5-{m}^2", kop.n, kop, mop, x0, y0, cfg, dict(grid=m, seed=seed))


def config4(seed: int = DEFAULT_SEED, n: int = 16384, rank: int = 512, nnull: int = 64,
            solve_factory=None) -> Problem:
    """solve_factory(M dense) -> callable b -> M^-1 b (GPU CG on a box); default LAPACK."""
    rng = np.random.default_rng(seed)
    eps = rng.uniform(1.0, 20.0, n)
    v = rng.standard_normal((n, rank)) * np.sqrt(1.0 / n)
    w = rng.standard_normal((n, rank)) * np.sqrt(0.5 / n)
    nbasis, _ = np.linalg.qr(rng.standard_normal((n, nnull)))
    a = v @ v.T
    a[np.diag_indices(n)] += eps
    b = w @ w.T
    amb = a - b
    # K = Pi (A - B) Pi with Pi = I - N N^T
    t = amb - nbasis @ (nbasis.T @ amb)
    k = t - (t @ nbasis) @ nbasis.T
    del t, amb
    mm = a + b
    del a, b
    # (A + A^T)/2 is exactly symmetric in floating point (x + y == y + x)
    k = np.asfortranarray(0.5 * (k + k.T))
    mm = np.asfortranarray(0.5 * (mm + mm.T))
    x_raw = np.asfortranarray(nbasis)
    y_raw = solve_factory(mm)(x_raw) if solve_factory else np.linalg.solve(mm, x_raw)
    x0, y0 = normalize_nullspace(x_raw, y_raw)
    cfg = dict(nev=32, nb=64, tol=1e-8)
    return Problem(f"config4-dense-n{n}", n, k, mm, x0, y0, cfg, dict(seed=seed))


def random_spd(n: int, cond: float, seed: int) -> np.ndarray:
    """Q^T D Q with log-uniform D spanning cond (SPEC.md make_random_spd_problem)."""
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    d = np.exp(rng.uniform(0.0, np.log(cond), n)) if cond > 1 else np.ones(n)
    a = (q * d) @ q.T
    il = np.tril_indices(n, -1)
    a.T[il] = a[il]
    return np.asfortranarray(a)
