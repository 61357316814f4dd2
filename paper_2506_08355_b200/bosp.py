"""Python mirror of the reference's BOSP API (proj/include/bosp/...), bound to the B200 C ABI.

Same names and argument meaning as the reference's C++ surface so tests read like the
reference's own:  LinearOperator.from_dense / from_csr / from_callback / identity /
scaled_identity / diagonal / shifted (+ stencil, new), InnerProduct, BospConfig,
GeneralizedNullspace, solve(K, M, ip, cfg, ns), block_inner / block_product / block_axpy,
mgs_biorth / cgs_biorth / biorth_against / biorth_residual, cg_solve, solve_small_lrep,
jacobi_svd, cholesky_lower, regression_coefficients, analytic_nullspace_T, compute_nullspace.
Every numeric call runs through libbosp_b200.so on the GPU (host small algebra excepted, as in
the north star); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from ._lib import (BospError, ContractViolation, CudaError, DegenerateSpectrum,  # noqa: F401
                   IngestionError, InitializationFailure, InvalidNullspace, NotEnoughSamples,
                   NullspaceLeak, NumericalAbort, RankMismatch, check, lib)


def _f(a, ndim=2):
    a = np.asarray(a, dtype=np.float64)
    if ndim == 2 and a.ndim == 1:
        a = a[:, None]
    return np.asfortranarray(a)


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _stencil_spec(nx, ny, nz, bc, scale, potential="none", origin=0.0, h=1.0, v=None, s0=0, s_global=0,
                  nz_global=0):
    bcs = {"neumann": 0, "dirichlet": 1}[bc]
    pot = {"none": 0, "harmonic": 1, "array": 2}[potential]
    vv = None if v is None else np.ascontiguousarray(v, dtype=np.float64)
    spec = L.Stencil(nx, ny, nz, bcs, scale, pot, origin, h, None if vv is None else vv.ctypes.data,
                     s0, s_global, nz_global)
    return spec, vv


class LinearOperator:
    """Apply-only operator (linear_operator.hpp:15-48); data lives in HBM."""
    dense, sparse_csr, matrix_free_callback = 0, 1, 2

    def __init__(self, handle, keep=None):
        self._h = handle
        self._keep = keep

    def __del__(self):
        try:
            if self._h:
                lib().bosp_op_free(self._h)
        except Exception:
            pass

    @classmethod
    def _make(cls, fn, *args, keep=None):
        h = L.OpPtr()
        check(fn(*args, C.byref(h)))
        return cls(h, keep)

    @classmethod
    def from_dense(cls, a):
        a = _f(a)
        if a.shape[0] != a.shape[1]:
            raise ContractViolation("LinearOperator: dense operator must be square")
        return cls._make(lib().bosp_op_dense, C.c_int64(a.shape[0]), _p(a))

    @classmethod
    def from_csr(cls, rowptr, colidx=None, vals=None):
        if colidx is None:  # problems.Csr
            rowptr, colidx, vals = rowptr.rowptr, rowptr.colidx, rowptr.vals
        rp = np.ascontiguousarray(rowptr, dtype=np.int64)
        ci = np.ascontiguousarray(colidx, dtype=np.int64)
        vv = np.ascontiguousarray(vals, dtype=np.float64)
        return cls._make(lib().bosp_op_csr, C.c_int64(rp.shape[0] - 1), _p(rp), _p(ci), _p(vv))

    @classmethod
    def from_matrix_market(cls, path):
        """Matrix Market file (coordinate real general|symmetric) -> device CSR operator."""
        return cls._make(lib().bosp_op_matrix_market, str(path).encode())

    @classmethod
    def from_callback(cls, dim, fn):
        """fn(x) -> y on (n, m) float64 arrays (host ApplyFn, linear_operator.cpp:45-47)."""
        def tramp(ctx, xp, yp, n, m):
            x = np.ctypeslib.as_array(xp, shape=(m, n)).T
            y = np.ctypeslib.as_array(yp, shape=(m, n)).T
            y[...] = fn(np.array(x))
        cb = L.HOST_APPLY(tramp)
        return cls._make(lib().bosp_op_callback, C.c_int64(dim), cb, None, keep=cb)

    @classmethod
    def from_device_callback(cls, dim, fn):
        """Device matrix-free plugin (bosp_op_device_callback): fn(device, x_ptr, ldx, y_ptr, ldy,
        n, ncols, stream_ptr) -> int status, called with HBM pointers of column-major blocks
        and the solver's cudaStream_t; it must enqueue y(:, j) = A x(:, j) on that stream and
        return 0 (nonzero aborts the solve).  The device analog of from_callback
        (linear_operator.hpp:19,25)."""
        def tramp(ctx, dev, xp, ldx, yp, ldy, n, m, stream):
            try:
                return int(fn(dev, xp or 0, ldx, yp or 0, ldy, n, m, stream or 0))
            except Exception:  # an exception must not unwind through C frames
                return -1
        cb = L.DEVICE_APPLY(tramp)
        return cls._make(lib().bosp_op_device_callback, C.c_int64(dim), cb, None, keep=cb)

    @classmethod
    def stencil(cls, nx, ny, nz, bc, scale, potential="none", origin=0.0, h=1.0, v=None,
                s0=0, s_global=0, nz_global=0):
        """Matrix-free stencil.  s_global > 0: this rank's slab of slow-axis planes
        [s0, s0 + nz) (3-D; grid rows for 2-D) out of s_global, under an attached communicator."""
        spec, vv = _stencil_spec(nx, ny, nz, bc, scale, potential, origin, h, v, s0, s_global, nz_global)
        return cls._make(lib().bosp_op_stencil, C.byref(spec), keep=vv)

    @classmethod
    def from_csr_rows(cls, n_global, row0, rowptr, colidx, vals):
        """Rows [row0, row0 + n_local) of a global CSR operator (global column indices); rowptr
        may keep the global offsets.  Needs an attached communicator (comm_init_nccl)."""
        rp = np.ascontiguousarray(rowptr, dtype=np.int64)
        ci = np.ascontiguousarray(colidx, dtype=np.int64)
        vv = np.ascontiguousarray(vals, dtype=np.float64)
        return cls._make(lib().bosp_op_csr_rows, C.c_int64(n_global), C.c_int64(row0),
                         C.c_int64(rp.shape[0] - 1), _p(rp), _p(ci), _p(vv))

    @classmethod
    def from_dense_rows(cls, n_global, row0, a_rows):
        """Rows [row0, row0 + n_local) of a dense n_global x n_global operator (n_local x n_global)."""
        a = _f(a_rows)
        if a.shape[1] != n_global:
            raise ContractViolation("from_dense_rows: a_rows must have n_global columns")
        return cls._make(lib().bosp_op_dense_rows, C.c_int64(n_global), C.c_int64(row0),
                         C.c_int64(a.shape[0]), _p(a))

    @classmethod
    def from_stencil(cls, s):
        """problems.Stencil -> matrix-free device operator."""
        return cls.stencil(s.nx, s.ny, s.nz, s.bc, s.scale, s.potential, s.origin, s.h, s.v)

    @classmethod
    def identity(cls, n):
        return cls._make(lib().bosp_op_identity, C.c_int64(n))

    @classmethod
    def scaled_identity(cls, n, alpha):
        return cls._make(lib().bosp_op_scaled_identity, C.c_int64(n), C.c_double(alpha))

    @classmethod
    def diagonal(cls, d):
        d = np.ascontiguousarray(d, dtype=np.float64)
        return cls._make(lib().bosp_op_diagonal, C.c_int64(d.shape[0]), _p(d))

    @classmethod
    def shifted(cls, a, sigma):
        return cls._make(lib().bosp_op_shifted, a._h, C.c_double(sigma), keep=a)

    @property
    def dim(self):
        return int(lib().bosp_op_dim(self._h))

    @property
    def kind(self):
        return int(lib().bosp_op_kind(self._h))

    def apply(self, x):
        x = _f(x)
        if x.shape[0] != self.dim:
            raise ContractViolation("LinearOperator::apply: dimension mismatch")
        y = np.zeros_like(x, order="F")
        check(lib().bosp_op_apply(self._h, C.c_int64(x.shape[1]), _p(x), _p(y)))
        return y


def block_apply(op, x):
    return op.apply(x)


class InnerProduct:
    """x^T B y (inner_product.hpp:12-29); identity when weight is None."""

    def __init__(self, weight: LinearOperator | None = None):
        self.weight = weight

    @property
    def weighted(self):
        return self.weight is not None

    def _h(self):
        return None if self.weight is None else self.weight._h


@dataclass
class BospConfig:  # bosp_solver.hpp:15-34
    nev: int = 1
    nb: int = 0
    tol: float = 1e-8
    ngs: int = 1
    s: int = 3
    moving: bool | None = None
    max_outer_iter: int = 500
    rng_seed: int = 0
    inner_cg_tol: float = 1e-2
    inner_cg_max_iter: int = 20
    tol_null: float = 1e-10
    rank_hint: int | None = None

    def c(self):
        return L.Config(self.nev, self.nb, self.tol, self.ngs, self.s,
                        -1 if self.moving is None else int(bool(self.moving)), self.max_outer_iter,
                        self.rng_seed, self.inner_cg_tol, self.inner_cg_max_iter, self.tol_null,
                        -1 if self.rank_hint is None else int(self.rank_hint))

    def effective_nb(self):
        if self.nb > 0:
            return min(self.nb, self.nev)
        return max(1, min((self.nev + 4) // 5, 150))

    def effective_moving(self):
        return bool(self.moving) if self.moving is not None else self.nev > 3 * self.effective_nb()


@dataclass
class GeneralizedNullspace:  # nullspace.hpp:13-19
    x0: np.ndarray
    y0: np.ndarray

    @property
    def r(self):
        return 0 if self.x0 is None else int(self.x0.shape[1])


@dataclass
class EigenResult:  # bosp_solver.hpp:71-81
    lambdas: np.ndarray
    x: np.ndarray
    y: np.ndarray
    iterations: int
    residuals: np.ndarray
    history: np.ndarray
    converged: bool
    nev_converged: int
    stats: dict = field(default_factory=dict)


class _Pinned:
    """Owner of a page-locked host buffer (bosp_host_alloc / cudaMallocHost)."""

    def __init__(self, nbytes):
        lib().bosp_host_alloc.restype = C.c_void_p
        self.ptr = lib().bosp_host_alloc(C.c_int64(max(int(nbytes), 8)))
        if not self.ptr:
            raise CudaError("bosp_host_alloc failed")

    def __del__(self):
        try:
            lib().bosp_host_free(C.c_void_p(self.ptr))
        except Exception:
            pass


def pinned_empty(shape, order="F"):
    """float64 array in page-locked host memory: eigenvector outputs written by DMA straight
    from HBM (no staging through the pinned ring)."""
    shape = tuple(int(v) for v in shape)
    count = int(np.prod(shape))
    owner = _Pinned(8 * count)
    buf = (C.c_double * max(count, 1)).from_address(owner.ptr)
    arr = np.frombuffer(buf, dtype=np.float64, count=count).reshape(shape, order=order)
    return _PinnedArray(arr, owner)


class _PinnedArray(np.ndarray):
    def __new__(cls, arr, owner):
        obj = arr.view(cls)
        obj._owner = owner
        return obj

    def __array_finalize__(self, obj):
        self._owner = getattr(obj, "_owner", None)


def solve(K: LinearOperator, M: LinearOperator, ip: InnerProduct | None, cfg: BospConfig,
          ns: GeneralizedNullspace | None = None, want_vectors=True, history_cap=2000,
          out=None) -> EigenResult:
    """bosp::solve (bosp_solver.cpp:513-536) on the B200.  out=(x, y): caller-owned n x nev
    Fortran-order float64 buffers for the eigenvectors (e.g. pinned_empty), reused across calls."""
    ip = ip or InnerProduct()
    n = K.dim
    cap = cfg.nev
    lam = np.zeros(cap)
    res = np.zeros(cap)
    if out is not None:
        x, y = out
        for a in (x, y):
            if a.shape != (n, cap) or a.dtype != np.float64 or not a.flags.f_contiguous:
                raise ContractViolation("solve: out buffers must be n x nev float64, column-major")
    else:
        x = np.zeros((n, cap), order="F") if want_vectors else None
        y = np.zeros((n, cap), order="F") if want_vectors else None
    hist = np.zeros((history_cap, cfg.nev))
    hrows, nout = C.c_int64(), C.c_int64()
    st = L.Stats()
    cc = cfg.c()
    if ns is None:
        r, x0, y0 = -1, None, None
    else:
        x0, y0 = _f(ns.x0), _f(ns.y0)
        r = x0.shape[1]
    check(lib().bosp_solve(K._h, M._h, ip._h(), C.byref(cc), C.c_int64(r), _p(x0), _p(y0),
                           C.c_int64(cap), _p(lam), _p(x), _p(y), _p(res), C.byref(nout),
                           C.byref(st), _p(hist), C.c_int64(history_cap), C.byref(hrows)))
    k = nout.value
    stats = {f[0]: getattr(st, f[0]) for f in L.Stats._fields_}
    return EigenResult(lam[:k], None if x is None else x[:, :k], None if y is None else y[:, :k],
                       int(st.iterations), res[:k], hist[:min(hrows.value, history_cap)],
                       bool(st.converged), int(st.nev_converged), stats)


def read_matrix_market(path):
    """read_matrix_market (matrix_market.cpp:26-91) -> problems.Csr (square) or the raw
    (rows, cols, rowptr, colidx, vals) tuple for rectangular files."""
    from .problems import Csr
    rows, cols, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    bp = str(path).encode()
    check(lib().bosp_read_matrix_market(bp, C.byref(rows), C.byref(cols), C.byref(nnz), None, None, None))
    rp = np.zeros(rows.value + 1, dtype=np.int64)
    ci = np.zeros(nnz.value, dtype=np.int64)
    vv = np.zeros(nnz.value)
    check(lib().bosp_read_matrix_market(bp, C.byref(rows), C.byref(cols), C.byref(nnz), _p(rp), _p(ci), _p(vv)))
    if rows.value == cols.value:
        return Csr(rows.value, rp, ci, vv)
    return rows.value, cols.value, rp, ci, vv


# ---- row-partitioned ranks ---------------------------------------------------------------
def _same_nccl_as_torch():
    """Load torch's NCCL first (when torch is installed) so the library's dlopen reuses it."""
    try:
        import torch  # noqa: F401
    except Exception:
        pass


def comm_nccl_unique_id() -> bytes:
    """ncclGetUniqueId: rank 0 creates it and broadcasts the 128 bytes (e.g. torch.distributed)."""
    _same_nccl_as_torch()
    buf = (C.c_ubyte * 128)()
    check(lib().bosp_comm_nccl_unique_id(buf))
    return bytes(buf)


def comm_init_nccl(uid: bytes, nranks: int, rank: int, n_global: int, row0: int):
    """Attach an NCCL communicator and this rank's row window [row0, ...) to the calling thread;
    afterwards solve() on partitioned operators returns this rank's rows of x, y."""
    _same_nccl_as_torch()
    buf = (C.c_ubyte * 128).from_buffer_copy(uid)
    check(lib().bosp_comm_init_nccl(buf, C.c_int32(nranks), C.c_int32(rank), C.c_int64(n_global),
                                    C.c_int64(row0)))


def comm_free():
    check(lib().bosp_comm_free())


def row_slice(op, nranks, rank):
    """Rows (row0, n_local) and slow-axis planes (s0, count) of one rank; the rule the native
    driver uses (multi.cpp row_slice): balanced rows, or balanced z-planes / grid rows."""
    from .problems import Stencil
    if isinstance(op, Stencil):
        three = op.nz > 1
        sg = op.nz if three else op.ny
        plane = op.nx * op.ny if three else op.nx
        s0 = sg * rank // nranks
        cnt = sg * (rank + 1) // nranks - s0
        return s0 * plane, cnt * plane, s0, cnt
    n = op.n if hasattr(op, "n") and not isinstance(op, np.ndarray) else np.asarray(op).shape[0]
    r0 = n * rank // nranks
    return r0, n * (rank + 1) // nranks - r0, 0, 0


def local_operator(op, nranks, rank):
    """This rank's LinearOperator slice of a global problems.Csr / problems.Stencil / dense array."""
    from .problems import Csr, Stencil
    row0, nl, s0, cnt = row_slice(op, nranks, rank)
    if isinstance(op, Stencil):
        three = op.nz > 1
        v = None if op.v is None else np.asarray(op.v)[row0:row0 + nl]
        return LinearOperator.stencil(op.nx, op.ny if three else cnt, cnt if three else 1, op.bc, op.scale,
                                      op.potential, op.origin, op.h, v, s0=s0,
                                      s_global=op.nz if three else op.ny, nz_global=op.nz)
    if isinstance(op, Csr):
        rp = op.rowptr[row0:row0 + nl + 1]
        return LinearOperator.from_csr_rows(op.n, row0, rp, op.colidx[rp[0]:rp[-1]], op.vals[rp[0]:rp[-1]])
    a = np.asarray(op, dtype=np.float64)
    return LinearOperator.from_dense_rows(a.shape[0], row0, a[row0:row0 + nl])


def _global_op(op):
    from .problems import Csr, Stencil
    g = L.GlobalOp()
    keep = []
    if isinstance(op, Stencil):
        spec, vv = _stencil_spec(op.nx, op.ny, op.nz, op.bc, op.scale, op.potential, op.origin, op.h, op.v)
        g.kind, g.n, g.stencil = 2, op.n, spec
        keep.append(vv)
    elif isinstance(op, Csr):
        rp = np.ascontiguousarray(op.rowptr, dtype=np.int64)
        ci = np.ascontiguousarray(op.colidx, dtype=np.int64)
        vv = np.ascontiguousarray(op.vals, dtype=np.float64)
        g.kind, g.n, g.rowptr, g.colidx, g.vals = 1, op.n, rp.ctypes.data, ci.ctypes.data, vv.ctypes.data
        keep += [rp, ci, vv]
    else:
        a = _f(op)
        g.kind, g.n, g.dense = 0, a.shape[0], a.ctypes.data
        keep.append(a)
    return g, keep


def solve_multi(nranks, K, M, cfg: BospConfig, ns: GeneralizedNullspace | None = None, ngpus=0,
                want_vectors=True, B=None) -> EigenResult:
    """Row-partitioned solve: nranks ranks as threads of this process over ngpus devices
    (several may share one GPU).  K, M (and the inner-product weight B): global problems.Csr /
    problems.Stencil / dense arrays."""
    gk, kk = _global_op(K)
    gm, km = _global_op(M)
    gb, kb = _global_op(B) if B is not None else (None, None)
    n = gk.n
    cap = cfg.nev
    lam, res = np.zeros(cap), np.zeros(cap)
    x = np.zeros((n, cap), order="F") if want_vectors else None
    y = np.zeros((n, cap), order="F") if want_vectors else None
    nout, st, cc = C.c_int64(), L.Stats(), cfg.c()
    if ns is None:
        r, x0, y0 = -1, None, None
    else:
        x0, y0 = _f(ns.x0), _f(ns.y0)
        r = x0.shape[1]
    check(lib().bosp_solve_multi(C.c_int32(nranks), C.c_int32(ngpus), C.byref(gk), C.byref(gm),
                                 None if gb is None else C.byref(gb), C.byref(cc),
                                 C.c_int64(r), _p(x0), _p(y0), C.c_int64(cap), _p(lam), _p(x), _p(y), _p(res),
                                 C.byref(nout), C.byref(st)))
    del kk, km
    k = nout.value
    stats = {f[0]: getattr(st, f[0]) for f in L.Stats._fields_}
    return EigenResult(lam[:k], None if x is None else x[:, :k], None if y is None else y[:, :k],
                       int(st.iterations), res[:k], np.zeros((0, cfg.nev)),
                       bool(st.converged), int(st.nev_converged), stats)


def regression_coefficients(history, idx, tol):
    h = np.ascontiguousarray(history, dtype=np.float64)
    a, b, d = C.c_double(), C.c_double(), C.c_int32()
    check(lib().bosp_regression(_p(h), C.c_int64(h.shape[0]), C.c_int64(h.shape[1]),
                                C.c_int64(idx), C.c_double(tol), C.byref(a), C.byref(b), C.byref(d)))
    return a.value, b.value, bool(d.value)


def analytic_nullspace_T(n):
    x0 = np.zeros((n, 1), order="F")
    y0 = np.zeros((n, 1), order="F")
    check(lib().bosp_analytic_nullspace_T(C.c_int64(n), _p(x0), _p(y0)))
    return GeneralizedNullspace(x0, y0)


def compute_nullspace(K, M, rank_hint=None, tol_null=1e-10, ip=None, seed=777, cap=256):
    n = K.dim
    x0 = np.zeros((n, cap), order="F")
    y0 = np.zeros((n, cap), order="F")
    r = C.c_int64()
    ip = ip or InnerProduct()
    check(lib().bosp_compute_nullspace(K._h, M._h, ip._h(), C.c_int64(-1 if rank_hint is None else rank_hint),
                                       C.c_double(tol_null), C.c_uint64(seed), C.c_int64(cap),
                                       C.byref(r), _p(x0), _p(y0)))
    return GeneralizedNullspace(x0[:, :r.value].copy(order="F"), y0[:, :r.value].copy(order="F"))


# ---- block kernels (kernels.hpp / biorth.hpp / cg.hpp) -------------------------------------
def block_inner(ip, x, y):
    x, y = _f(x), _f(y)
    if x.shape[0] != y.shape[0]:
        raise ContractViolation("block_inner: dimension mismatch")
    ip = ip or InnerProduct()
    g = np.zeros((x.shape[1], y.shape[1]), order="F")
    check(lib().bosp_block_inner(ip._h(), C.c_int64(x.shape[0]), C.c_int64(x.shape[1]),
                                 C.c_int64(y.shape[1]), _p(x), _p(y), _p(g)))
    return g


def _test_gram_jobs(x, y, nseg=1, njobs=3):
    """Test hook: the solver's multi-job Gram launch -> (XᵀY, XᵀX, YᵀY); X in nseg segments."""
    x, y = _f(x), _f(y)
    n, a, b = x.shape[0], x.shape[1], y.shape[1]
    out = np.zeros(a * b + a * a + b * b)
    check(lib().bosp_test_gram_jobs(C.c_int64(n), C.c_int64(a), C.c_int64(b), _p(x), _p(y), C.c_int32(nseg),
                                    C.c_int32(njobs), _p(out)))
    return (out[:a * b].reshape((a, b), order="F"), out[a * b:a * b + a * a].reshape((a, a), order="F"),
            out[a * b + a * a:].reshape((b, b), order="F"))


def _test_gram_sym(x, y, same=True):
    """Test hook: symmetric Gram -> [X | Y]^T [X | Y] (same) or X^T Y via the mirrored path."""
    x, y = _f(x), _f(y)
    n, a = x.shape
    w = 2 * a if same else a
    out = np.zeros((w, w), order="F")
    check(lib().bosp_test_gram_sym(C.c_int64(n), C.c_int64(a), _p(x), _p(y), C.c_int32(1 if same else 0), _p(out)))
    return out


def _test_biorth_apply(x, y, a, b):
    """Test hook: the fused MGS-Biorth application -> (P = X A, Q = Y B, P^T Q)."""
    x, y, a, b = _f(x), _f(y), _f(a), _f(b)
    n, k, kb = x.shape[0], x.shape[1], a.shape[1]
    p = np.zeros((n, kb), order="F")
    q = np.zeros((n, kb), order="F")
    g = np.zeros((kb, kb), order="F")
    check(lib().bosp_test_biorth_apply(C.c_int64(n), C.c_int64(k), C.c_int64(kb), _p(x), _p(y), _p(a), _p(b),
                                       _p(p), _p(q), _p(g)))
    return p, q, g


def _test_mgs_dev(x, y):
    """Test hook: the solver's device MGS-Biorth -> (P, Q, second_pass) of the kept columns."""
    x, y = _f(x), _f(y)
    n, m = x.shape
    p = np.zeros((n, m), order="F")
    q = np.zeros((n, m), order="F")
    nk, sp = C.c_int64(), C.c_int32()
    check(lib().bosp_test_mgs_dev(C.c_int64(n), C.c_int64(m), _p(x), _p(y), _p(p), _p(q), C.byref(nk), C.byref(sp)))
    k = nk.value
    return p[:, :k].copy(order="F"), q[:, :k].copy(order="F"), bool(sp.value)


def block_product(x, c):
    x, c = _f(x), _f(c)
    if x.shape[1] != c.shape[0]:
        raise ContractViolation("block_product: shape mismatch")
    out = np.zeros((x.shape[0], c.shape[1]), order="F")
    check(lib().bosp_block_product(C.c_int64(x.shape[0]), C.c_int64(x.shape[1]),
                                   C.c_int64(c.shape[1]), _p(x), _p(c), _p(out)))
    return out


def block_axpy(x, c, y):
    x, c = _f(x), _f(c)
    y = np.array(y, dtype=np.float64, order="F", copy=True)
    if y.ndim == 1:
        y = y[:, None].copy(order="F")
    if x.shape[1] != c.shape[0] or c.shape[1] != y.shape[1] or x.shape[0] != y.shape[0]:
        raise ContractViolation("block_axpy: shape mismatch")
    check(lib().bosp_block_axpy(C.c_int64(x.shape[0]), C.c_int64(x.shape[1]),
                                C.c_int64(c.shape[1]), _p(x), _p(c), _p(y)))
    return y


def _biorth(x, y, ip, drop_tol, classical):
    x, y = _f(x), _f(y)
    if x.shape != y.shape:
        raise ContractViolation("biorth: X and Y must have equal shape")
    n, m = x.shape
    ip = ip or InnerProduct()
    p = np.zeros((n, m), order="F")
    q = np.zeros((n, m), order="F")
    kept = np.zeros(max(m, 1), dtype=np.int64)
    dropped = np.zeros(max(m, 1), dtype=np.int64)
    nk, nd = C.c_int64(), C.c_int64()
    check(lib().bosp_biorth(C.c_int32(int(classical)), ip._h(), C.c_int64(n), C.c_int64(m), _p(x),
                            _p(y), C.c_double(drop_tol), _p(p), _p(q), _p(kept), C.byref(nk),
                            _p(dropped), C.byref(nd)))
    k = nk.value
    return p[:, :k].copy(order="F"), q[:, :k].copy(order="F"), list(kept[:k]), list(dropped[:nd.value])


def mgs_biorth(x, y, ip=None, drop_tol=1e-12):
    """(P, Q, kept, dropped) -- biorth.cpp:102-109."""
    return _biorth(x, y, ip, drop_tol, False)


def cgs_biorth(x, y, ip=None, drop_tol=1e-12):
    return _biorth(x, y, ip, drop_tol, True)


def biorth_against(bases, x, y, ip=None):
    x, y = _f(x), _f(y)
    n, m = x.shape
    ip = ip or InnerProduct()
    if x.shape[0] != y.shape[0]:
        raise ContractViolation("biorth_against: X and Y dimension mismatch")
    ps = [_f(p) for p, _ in bases]
    qs = [_f(q) for _, q in bases]
    if any(p.shape[0] != n or q.shape != p.shape for p, q in zip(ps, qs)):
        raise ContractViolation("biorth_against: basis dimension mismatch")
    widths = np.array([p.shape[1] for p in ps] or [0], dtype=np.int64)
    parr = (C.c_void_p * max(1, len(ps)))(*[p.ctypes.data for p in ps])
    qarr = (C.c_void_p * max(1, len(qs)))(*[q.ctypes.data for q in qs])
    xo = np.zeros((n, m), order="F")
    yo = np.zeros((n, m), order="F")
    check(lib().bosp_biorth_against(ip._h(), C.c_int64(n), C.c_int64(len(ps)), _p(widths), parr,
                                    qarr, C.c_int64(m), _p(x), _p(y), _p(xo), _p(yo)))
    return xo, yo


def biorth_residual(p, q, ip=None):
    p, q = _f(p), _f(q)
    ip = ip or InnerProduct()
    out = C.c_double()
    check(lib().bosp_biorth_residual(ip._h(), C.c_int64(p.shape[0]), C.c_int64(p.shape[1]),
                                     _p(p), _p(q), C.byref(out)))
    return out.value


def cg_solve(op, rhs, x0=None, tol=1e-2, max_iter=20):
    rhs = _f(rhs)
    x0 = None if x0 is None else _f(x0)
    x = np.zeros_like(rhs, order="F")
    br, mi = C.c_int32(), C.c_int64()
    check(lib().bosp_cg_solve(op._h, C.c_int64(rhs.shape[1]), _p(rhs), _p(x0), C.c_double(tol),
                              C.c_int64(max_iter), _p(x), C.byref(br), C.byref(mi)))
    return x, bool(br.value), mi.value


def solve_small_lrep(khat, mhat, k):
    khat, mhat = _f(khat), _f(mhat)
    d = khat.shape[0]
    lam = np.zeros(k)
    xh = np.zeros((d, k), order="F")
    yh = np.zeros((d, k), order="F")
    check(lib().bosp_solve_small_lrep(C.c_int64(d), _p(khat), _p(mhat), C.c_int64(k), _p(lam),
                                      _p(xh), _p(yh)))
    return lam, xh, yh


def jacobi_svd(a):
    a = _f(a)
    m, k = a.shape
    u = np.zeros((m, k), order="F")
    v = np.zeros((k, k), order="F")
    s = np.zeros(k)
    sw, cv = C.c_int64(), C.c_int32()
    check(lib().bosp_jacobi_svd(C.c_int64(m), C.c_int64(k), _p(a), _p(u), _p(s), _p(v),
                                C.byref(sw), C.byref(cv)))
    return u, s, v, sw.value, bool(cv.value)


def cholesky_lower(a):
    a = _f(a)
    n = a.shape[0]
    l = np.zeros((n, n), order="F")
    ok = C.c_int32()
    check(lib().bosp_cholesky(C.c_int64(n), _p(a), _p(l), C.byref(ok)))
    return l if ok.value else None


def seed_blocks(seed, n, d):
    """(U, V) initial blocks as initialize() draws them, generated on the device."""
    u = np.zeros((n, d), order="F")
    v = np.zeros((n, d), order="F")
    check(lib().bosp_seed_blocks(C.c_uint64(seed), C.c_int64(n), C.c_int64(d), _p(u), _p(v)))
    return u, v


# ---- measurement hooks ----------------------------------------------------------------------
def device_info():
    buf = C.create_string_buffer(256)
    sms = lib().bosp_device_info(buf, 256)
    if sms < 0:
        check(-sms)
    return buf.value.decode(), sms


def profile_enable(family: str | None):
    lib().bosp_profile_enable((family or "").encode())


def profile_collect():
    n, ms, b, f = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
    rc, rb = C.c_int64(), C.c_double()
    lib().bosp_profile_collect_regions(C.byref(n), C.byref(ms), C.byref(b), C.byref(f),
                                       C.byref(rc), C.byref(rb))
    out = dict(launches=n.value, ms=ms.value, bytes=b.value, flops=f.value,
               region_calls=rc.value, region_bytes=rb.value)
    L_ = lib()
    L_.bosp_profile_family_report.restype = C.c_int64
    need = L_.bosp_profile_family_report(None, C.c_int64(0))
    buf = C.create_string_buffer(int(need))
    L_.bosp_profile_family_report(buf, C.c_int64(need))
    fams = {}
    for line in buf.value.decode().splitlines():
        f, l, m, by, fl = line.split()
        if f == "@region":
            out["region_flops"] = float(fl)
            continue
        fams[f] = dict(launches=int(l), ms=float(m), bytes=float(by), flops=float(fl))
    out["families"] = fams
    return out


def launch_count():
    return int(lib().bosp_launch_count())


def launch_reset():
    lib().bosp_launch_reset()


def launch_families():
    buf = C.create_string_buffer(4096)
    lib().bosp_launch_families(buf, 4096)
    out = {}
    for item in buf.value.decode().split(";"):
        if "=" in item:
            k, v = item.split("=")
            out[k] = int(v)
    return out


def device_sync():
    lib().bosp_device_sync()


def bench_apply(op, ncols, reps=20):
    ms = C.c_double()
    check(lib().bosp_bench_apply(op._h, C.c_int64(ncols), C.c_int64(reps), C.byref(ms)))
    return ms.value


def bench_cg(op, ncols, iters=20, reps=5):
    """Mean ms per batched-CG iteration (all columns active)."""
    ms = C.c_double()
    check(lib().bosp_bench_cg(op._h, C.c_int64(ncols), C.c_int64(iters), C.c_int64(reps), C.byref(ms)))
    return ms.value


def bench_blas(kind, n, a, b, reps=20):
    """kind: 'gram' | 'product' | 'axpy' -> mean ms per call on device-resident data."""
    k = {"gram": 0, "product": 1, "axpy": 2, "gram3": 3, "gramsym": 4, "mgsapply": 5, "mgs": 6, "mgs_cold": 7}[kind]
    ms = C.c_double()
    check(lib().bosp_bench_blas(C.c_int32(k), C.c_int64(n), C.c_int64(a), C.c_int64(b),
                                C.c_int64(reps), C.byref(ms)))
    return ms.value


def device_solver(op_or_problem_op, tol=1e-13, max_iter=20000):
    """b -> M^-1 b by the batched device CG (setup helper for the nullspace pair Y0 = M^-1 X0;
    M SPD).  Accepts a LinearOperator or a problems.{Csr,Stencil} / dense ndarray."""
    from . import problems as P
    op = op_or_problem_op
    if not isinstance(op, LinearOperator):
        if isinstance(op, np.ndarray):
            op = LinearOperator.from_dense(op)
        elif isinstance(op, P.Stencil):
            op = LinearOperator.from_stencil(op)
        else:
            op = LinearOperator.from_csr(op)

    def solve(b):
        x, _, _ = cg_solve(op, b, tol=tol, max_iter=max_iter)
        return x
    return solve


def operators_for(problem):
    """problems.Problem -> (K, M) device operators (dense / CSR / matrix-free stencil)."""
    from . import problems as P

    def one(op):
        if isinstance(op, np.ndarray):
            return LinearOperator.from_dense(op)
        if isinstance(op, P.Stencil):
            return LinearOperator.from_stencil(op)
        return LinearOperator.from_csr(op)
    return one(problem.K), one(problem.M)
