"""ORACLE / TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_ref/libbosp_ref.so.

The shared library is the UNMODIFIED reference (``/root/reference/proj/src``) compiled by
``oracle/Makefile`` plus our shim ``oracle/ref_shim.cpp``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / ``--impl reference``) may use
this module, and only as the checker or the CPU baseline -- never as the product path.

Operators are passed as plain numpy arrays:
  ("dense", A)                       -> LinearOperator::from_dense   (linear_operator.cpp:12-31)
  ("csr", (rowptr, colidx, vals))    -> LinearOperator::from_csr     (linear_operator.cpp:33-43)
  ("diag", d)                        -> LinearOperator::diagonal     (linear_operator.cpp:68-79)
  ("identity", n)                    -> LinearOperator::identity     (linear_operator.cpp:49-55)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libbosp_ref.so")

STATUS_NAMES = {
    0: "ok", 1: "ContractViolation", 2: "IngestionError", 3: "NullspaceLeak",
    4: "DegenerateSpectrum", 5: "RankMismatch", 6: "InvalidNullspace",
    7: "InitializationFailure", 8: "NotEnoughSamples", 9: "NumericalAbort", 11: "Error",
}


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS_NAMES.get(status, "Error")


class _OpDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int64), ("dense", C.c_void_p),
                ("rowptr", C.c_void_p), ("colidx", C.c_void_p), ("vals", C.c_void_p),
                ("nnz", C.c_int64)]


class _Config(C.Structure):
    _fields_ = [("nev", C.c_int64), ("nb", C.c_int64), ("tol", C.c_double),
                ("ngs", C.c_int64), ("s", C.c_int64), ("moving", C.c_int32),
                ("max_outer_iter", C.c_int64), ("rng_seed", C.c_uint64),
                ("inner_cg_tol", C.c_double), ("inner_cg_max_iter", C.c_int64),
                ("tol_null", C.c_double), ("rank_hint", C.c_int64)]


class _Stats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("matvec_count", C.c_int64),
                ("step3_matvecs", C.c_int64), ("step3_vecprods", C.c_int64),
                ("max_width_u", C.c_int64), ("max_biorth_deviation", C.c_double),
                ("max_deflation_crossgram", C.c_double), ("final_biorth_deviation", C.c_double),
                ("nevconv_monotone", C.c_int32), ("wall_seconds", C.c_double),
                ("nev_converged", C.c_int64), ("converged", C.c_int32)]


_lib = None


def use_library(path: str | None):
    """Bind this module to another build of ref_shim.cpp -- tests/test_compat.py compiles the
    same shim against the B200 library's reference-compatible headers and drives it through
    these very wrappers.  None restores oracle/_ref."""
    global _lib, LIB_PATH
    LIB_PATH = path or os.path.join(_HERE, "_ref", "libbosp_ref.so")
    _lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle` (needs /root/reference)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_biorth_residual.argtypes = None
    return _lib


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _check(status: int):
    if status != 0:
        raise RefError(status, lib().ref_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _fortran(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


class _Op:
    """Keeps the numpy buffers of one operator descriptor alive."""

    def __init__(self, spec):
        kind, payload = spec
        self.keep = []
        d = _OpDesc()
        if kind == "dense":
            a = _fortran(payload)
            self.keep.append(a)
            d.kind, d.n, d.dense = 0, a.shape[0], a.ctypes.data
        elif kind == "csr":
            rp, ci, vv = payload
            rp = np.ascontiguousarray(rp, dtype=np.int64)
            ci = np.ascontiguousarray(ci, dtype=np.int64)
            vv = _f64(vv)
            self.keep += [rp, ci, vv]
            d.kind, d.n = 1, rp.shape[0] - 1
            d.rowptr, d.colidx, d.vals, d.nnz = rp.ctypes.data, ci.ctypes.data, vv.ctypes.data, vv.shape[0]
        elif kind == "diag":
            v = _f64(payload)
            self.keep.append(v)
            d.kind, d.n, d.vals = 2, v.shape[0], v.ctypes.data
        elif kind == "identity":
            d.kind, d.n = 3, int(payload)
        else:
            raise ValueError(kind)
        self.desc = d
        self.n = d.n

    def ref(self):
        return C.byref(self.desc)


def _opt(spec):
    return None if spec is None else _Op(spec)


@dataclass
class RefConfig:
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

    def c(self) -> _Config:
        return _Config(self.nev, self.nb, self.tol, self.ngs, self.s,
                       -1 if self.moving is None else int(bool(self.moving)),
                       self.max_outer_iter, self.rng_seed, self.inner_cg_tol,
                       self.inner_cg_max_iter, self.tol_null,
                       -1 if self.rank_hint is None else self.rank_hint)


@dataclass
class RefResult:
    lambdas: np.ndarray
    x: np.ndarray
    y: np.ndarray
    residuals: np.ndarray
    stats: dict
    history: np.ndarray = field(default=None)


def set_threads(n: int):
    lib().ref_set_threads(int(n))


def threads() -> int:
    return int(lib().ref_threads())


def solve(K, M, cfg: RefConfig, ns=None, B=None, want_vectors=True, history_cap=1000) -> RefResult:
    k, m, b = _Op(K), _Op(M), _opt(B)
    n = k.n
    nev = cfg.nev
    lam = np.zeros(nev)
    res = np.zeros(nev)
    x = np.zeros((n, nev), order="F") if want_vectors else None
    y = np.zeros((n, nev), order="F") if want_vectors else None
    hist = np.zeros((history_cap, nev))
    hrows = C.c_int64(0)
    nout = C.c_int64(0)
    st = _Stats()
    cfgc = cfg.c()
    if ns is not None:
        x0, y0 = _fortran(ns[0]), _fortran(ns[1])
        r = x0.shape[1]
        have = 1
    else:
        x0 = y0 = np.zeros((n, 0), order="F")
        r, have = 0, 0
    _check(lib().ref_solve(k.ref(), m.ref(), None if b is None else b.ref(), C.byref(cfgc),
                           C.c_int32(have), C.c_int64(r), _p(x0), _p(y0), _p(lam),
                           _p(x), _p(y), _p(res), C.byref(nout), C.byref(st), _p(hist),
                           C.c_int64(history_cap), C.byref(hrows)))
    no = nout.value
    stats = {f[0]: getattr(st, f[0]) for f in _Stats._fields_}
    return RefResult(lam[:no], None if x is None else x[:, :no], None if y is None else y[:, :no],
                     res[:no], stats, hist[:min(hrows.value, history_cap)])


def time_iterations(K, M, cfg: RefConfig, ns, k_iters: int, B=None):
    k, m, b = _Op(K), _Op(M), _opt(B)
    x0, y0 = _fortran(ns[0]), _fortran(ns[1])
    t_init, t_it = C.c_double(), C.c_double()
    done, conv, nevc = C.c_int64(), C.c_int32(), C.c_int64()
    cfgc = cfg.c()
    _check(lib().ref_time_iterations(k.ref(), m.ref(), None if b is None else b.ref(),
                                     C.byref(cfgc), C.c_int64(x0.shape[1]), _p(x0), _p(y0),
                                     C.c_int64(k_iters), C.byref(t_init), C.byref(t_it),
                                     C.byref(done), C.byref(conv), C.byref(nevc)))
    return dict(t_init=t_init.value, t_iters=t_it.value, iters=done.value,
                converged=bool(conv.value), nev_conv=nevc.value)


def read_matrix_market(path: str):
    """The reference's read_matrix_market (matrix_market.cpp:26-91) -> (rows, cols, rowptr,
    colidx, vals) as int64 / float64 arrays."""
    rows, cols, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    bp = str(path).encode()
    _check(lib().ref_read_matrix_market(bp, C.byref(rows), C.byref(cols), C.byref(nnz), None, None, None))
    rp = np.zeros(rows.value + 1, dtype=np.int64)
    ci = np.zeros(nnz.value, dtype=np.int64)
    vv = np.zeros(nnz.value)
    _check(lib().ref_read_matrix_market(bp, C.byref(rows), C.byref(cols), C.byref(nnz), _p(rp), _p(ci), _p(vv)))
    return rows.value, cols.value, rp, ci, vv


def fill_uniform(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count)
    _check(lib().ref_fill_uniform(C.c_uint64(seed), C.c_int64(count), _p(out)))
    return out


def op_apply(A, x):
    a = _Op(A)
    x = _fortran(x if x.ndim == 2 else x[:, None])
    y = np.zeros_like(x, order="F")
    _check(lib().ref_op_apply(a.ref(), C.c_int64(x.shape[1]), _p(x), _p(y)))
    return y


def block_inner(x, y, B=None):
    x, y = _fortran(x), _fortran(y)
    b = _opt(B)
    g = np.zeros((x.shape[1], y.shape[1]), order="F")
    _check(lib().ref_block_inner(None if b is None else b.ref(), C.c_int64(x.shape[0]),
                                 C.c_int64(x.shape[1]), C.c_int64(y.shape[1]), _p(x), _p(y), _p(g)))
    return g


def block_product(x, c):
    x, c = _fortran(x), _fortran(c)
    out = np.zeros((x.shape[0], c.shape[1]), order="F")
    _check(lib().ref_block_product(C.c_int64(x.shape[0]), C.c_int64(x.shape[1]),
                                   C.c_int64(c.shape[1]), _p(x), _p(c), _p(out)))
    return out


def block_axpy(x, c, y):
    x, c = _fortran(x), _fortran(c)
    y = np.array(y, dtype=np.float64, order="F", copy=True)
    _check(lib().ref_block_axpy(C.c_int64(x.shape[0]), C.c_int64(x.shape[1]),
                                C.c_int64(c.shape[1]), _p(x), _p(c), _p(y)))
    return y


def biorth(x, y, drop_tol=1e-12, classical=False, B=None):
    x, y = _fortran(x), _fortran(y)
    n, m = x.shape
    b = _opt(B)
    p = np.zeros((n, m), order="F")
    q = np.zeros((n, m), order="F")
    kept = np.zeros(m, dtype=np.int64)
    dropped = np.zeros(m, dtype=np.int64)
    nk, nd = C.c_int64(), C.c_int64()
    _check(lib().ref_biorth(C.c_int32(int(classical)), None if b is None else b.ref(),
                            C.c_int64(n), C.c_int64(m), _p(x), _p(y), C.c_double(drop_tol),
                            _p(p), _p(q), _p(kept), C.byref(nk), _p(dropped), C.byref(nd)))
    k = nk.value
    return p[:, :k].copy(order="F"), q[:, :k].copy(order="F"), list(kept[:k]), list(dropped[:nd.value])


def mgs_biorth(x, y, drop_tol=1e-12, B=None):
    return biorth(x, y, drop_tol, False, B)


def cgs_biorth(x, y, drop_tol=1e-12, B=None):
    return biorth(x, y, drop_tol, True, B)


def biorth_against(bases, x, y, B=None):
    x, y = _fortran(x), _fortran(y)
    n, m = x.shape
    b = _opt(B)
    ps = [_fortran(p) for p, _ in bases]
    qs = [_fortran(q) for _, q in bases]
    widths = np.array([p.shape[1] for p in ps], dtype=np.int64)
    parr = (C.c_void_p * max(1, len(ps)))(*[p.ctypes.data for p in ps])
    qarr = (C.c_void_p * max(1, len(qs)))(*[q.ctypes.data for q in qs])
    xo = np.zeros((n, m), order="F")
    yo = np.zeros((n, m), order="F")
    _check(lib().ref_biorth_against(None if b is None else b.ref(), C.c_int64(n),
                                    C.c_int64(len(ps)), _p(widths), parr, qarr, C.c_int64(m),
                                    _p(x), _p(y), _p(xo), _p(yo)))
    return xo, yo


def biorth_residual(p, q, B=None):
    p, q = _fortran(p), _fortran(q)
    b = _opt(B)
    out = C.c_double()
    _check(lib().ref_biorth_residual(None if b is None else b.ref(), C.c_int64(p.shape[0]),
                                     C.c_int64(p.shape[1]), _p(p), _p(q), C.byref(out)))
    return out.value


def cg_solve(A, rhs, x0=None, tol=1e-2, max_iter=20):
    a = _Op(A)
    rhs = _fortran(rhs)
    x0 = np.zeros_like(rhs, order="F") if x0 is None else _fortran(x0)
    x = np.zeros_like(rhs, order="F")
    br, mi = C.c_int32(), C.c_int64()
    _check(lib().ref_cg_solve(a.ref(), C.c_int64(rhs.shape[1]), _p(rhs), _p(x0), C.c_double(tol),
                              C.c_int64(max_iter), _p(x), C.byref(br), C.byref(mi)))
    return x, bool(br.value), mi.value


def solve_small_lrep(khat, mhat, k):
    khat, mhat = _fortran(khat), _fortran(mhat)
    d = khat.shape[0]
    lam = np.zeros(k)
    xh = np.zeros((d, k), order="F")
    yh = np.zeros((d, k), order="F")
    _check(lib().ref_solve_small_lrep(C.c_int64(d), _p(khat), _p(mhat), C.c_int64(k), _p(lam),
                                      _p(xh), _p(yh)))
    return lam, xh, yh


def jacobi_svd(a):
    a = _fortran(a)
    m, k = a.shape
    u = np.zeros((m, k), order="F")
    v = np.zeros((k, k), order="F")
    s = np.zeros(k)
    sw, cv = C.c_int64(), C.c_int32()
    _check(lib().ref_jacobi_svd(C.c_int64(m), C.c_int64(k), _p(a), _p(u), _p(s), _p(v),
                                C.byref(sw), C.byref(cv)))
    return u, s, v, sw.value, bool(cv.value)


def cholesky(a):
    a = _fortran(a)
    n = a.shape[0]
    l = np.zeros((n, n), order="F")
    ok = C.c_int32()
    _check(lib().ref_cholesky(C.c_int64(n), _p(a), _p(l), C.byref(ok)))
    return l if ok.value else None


def spectral_norm(a):
    a = _fortran(a)
    out = C.c_double()
    _check(lib().ref_spectral_norm(C.c_int64(a.shape[0]), C.c_int64(a.shape[1]), _p(a),
                                   C.byref(out)))
    return out.value


def compute_nullspace(K, M, rank_hint=None, tol_null=1e-10, seed=777, B=None, cap=128):
    k, m, b = _Op(K), _Op(M), _opt(B)
    n = k.n
    x0 = np.zeros((n, cap), order="F")
    y0 = np.zeros((n, cap), order="F")
    r = C.c_int64()
    _check(lib().ref_compute_nullspace(k.ref(), m.ref(), None if b is None else b.ref(),
                                       C.c_int64(-1 if rank_hint is None else rank_hint),
                                       C.c_double(tol_null), C.c_uint64(seed), C.c_int64(cap),
                                       C.byref(r), _p(x0), _p(y0)))
    return x0[:, :r.value].copy(order="F"), y0[:, :r.value].copy(order="F")


def analytic_nullspace_T(n):
    x0 = np.zeros((n, 1), order="F")
    y0 = np.zeros((n, 1), order="F")
    _check(lib().ref_analytic_nullspace_T(C.c_int64(n), _p(x0), _p(y0)))
    return x0, y0


def regression_coefficients(history, idx, tol):
    h = np.ascontiguousarray(history, dtype=np.float64)
    a, b, dg = C.c_double(), C.c_double(), C.c_int32()
    _check(lib().ref_regression(_p(h), C.c_int64(h.shape[0]), C.c_int64(h.shape[1]),
                                C.c_int64(idx), C.c_double(tol), C.byref(a), C.byref(b),
                                C.byref(dg)))
    return a.value, b.value, bool(dg.value)
