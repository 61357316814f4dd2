"""ORACLE / TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference BOSP solver.

This is the CPU checker for the B200 path, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline leg may import it.  Each function
restates one reference function (file:line relative to /root/reference/proj) with the same
control flow and thresholds; n-length arithmetic is vectorised with numpy, so the summation
order (and hence the last bits) differ from the reference's serial loops.  The restatement is
pinned against the reference itself (oracle/_ref, built from the unmodified sources) and the
paper's published tables by ``tests/test_oracle.py``.

Operators are callables ``apply(X) -> A @ X`` on (n, m) float64 arrays (column-major not
required here).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------------------------
# RNG: std::mt19937_64 + std::uniform_real_distribution<double>(-1, 1) as libstdc++ draws them
# (block_vectors.cpp:27-30).  Published MT19937-64 algorithm (Matsumoto & Nishimura, 2004);
# generate_canonical<double, 53> consumes one 64-bit draw: u = double(x) / 2^64.
# ----------------------------------------------------------------------------------------------
_NN, _MM = 312, 156
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)
_UM = np.uint64(0xFFFFFFFF80000000)
_LM = np.uint64(0x7FFFFFFF)


class MT19937_64:
    def __init__(self, seed: int):
        mt = [0] * _NN
        mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, _NN):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.mt = np.array(mt, dtype=np.uint64)
        self.buf = np.zeros(0, dtype=np.uint64)

    def _twist(self):
        mt = self.mt
        one = np.uint64(1)
        # i in [0, NN-MM): uses old mt[i+1], old mt[i+MM]
        x = (mt[0:_NN - _MM] & _UM) | (mt[1:_NN - _MM + 1] & _LM)
        mt[0:_NN - _MM] = mt[_MM:_NN] ^ (x >> one) ^ np.where(x & one, _MATRIX_A, np.uint64(0))
        # i in [NN-MM, NN-1): uses old mt[i+1], new mt[i+MM-NN]
        for lo in range(_NN - _MM, _NN - 1, _MM):
            hi = min(lo + _MM, _NN - 1)
            x = (mt[lo:hi] & _UM) | (mt[lo + 1:hi + 1] & _LM)
            mt[lo:hi] = mt[lo + _MM - _NN:hi + _MM - _NN] ^ (x >> one) ^ np.where(x & one, _MATRIX_A, np.uint64(0))
        x = (mt[_NN - 1] & _UM) | (mt[0] & _LM)
        mt[_NN - 1] = mt[_MM - 1] ^ (x >> one) ^ (_MATRIX_A if int(x) & 1 else np.uint64(0))
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        return y

    def draw(self, count: int) -> np.ndarray:
        parts = [self.buf]
        have = self.buf.shape[0]
        while have < count:
            blk = self._twist()
            parts.append(blk)
            have += blk.shape[0]
        allv = np.concatenate(parts)
        self.buf = allv[count:]
        return allv[:count]

    def uniform(self, count: int, a: float = -1.0, b: float = 1.0) -> np.ndarray:
        u = self.draw(count).astype(np.float64) / 18446744073709551616.0
        u = np.where(u >= 1.0, np.nextafter(1.0, 0.0), u)
        return u * (b - a) + a


def fill_uniform(rng: MT19937_64, n: int, m: int) -> np.ndarray:
    """BlockVectors::fill_uniform (block_vectors.cpp:27-30), column-major fill."""
    return rng.uniform(n * m).reshape((m, n)).T.copy()


# ----------------------------------------------------------------------------------------------
# Errors (errors.hpp:9-69)
# ----------------------------------------------------------------------------------------------
class Error(RuntimeError):
    pass


class ContractViolation(Error):
    pass


class NullspaceLeak(Error):
    pass


class DegenerateSpectrum(Error):
    pass


class InitializationFailure(Error):
    pass


class NotEnoughSamples(Error):
    pass


class NumericalAbort(Error):
    pass


# ----------------------------------------------------------------------------------------------
# Block kernels (kernels.cpp:47-104) and the inner product (inner_product.cpp:11-32)
# ----------------------------------------------------------------------------------------------
class InnerProduct:
    def __init__(self, weight=None):
        self.weight = weight

    @property
    def weighted(self):
        return self.weight is not None

    def apply_weight(self, y):
        return y.copy() if self.weight is None else self.weight(y)

    def dot(self, x, y):
        if self.weight is None:
            return float(x @ y)
        return float(x @ self.weight(y[:, None])[:, 0])

    def norm(self, x):
        return math.sqrt(max(0.0, self.dot(x, x)))


def block_inner(ip: InnerProduct, x, y):
    """G[i, j] = <x_i, y_j> under ip; Y <- B Y first (kernels.cpp:47-68)."""
    if x.shape[0] != y.shape[0]:
        raise ContractViolation("block_inner: dimension mismatch")
    rhs = ip.apply_weight(y) if ip.weighted else y
    return x.T @ rhs


def block_product(x, c):
    """X C (kernels.cpp:70-87)."""
    if x.shape[1] != c.shape[0]:
        raise ContractViolation("block_product: shape mismatch")
    return x @ c


def block_axpy(x, c, y):
    """Y - X C (kernels.cpp:89-104)."""
    if x.shape[1] != c.shape[0] or c.shape[1] != y.shape[1] or x.shape[0] != y.shape[0]:
        raise ContractViolation("block_axpy: shape mismatch")
    return y - x @ c


# ----------------------------------------------------------------------------------------------
# Per-column CG (cg.cpp:11-58)
# ----------------------------------------------------------------------------------------------
def cg_solve(op, rhs, x0, tol, max_iter):
    x = x0.copy()
    breakdown = False
    max_used = 0
    for j in range(rhs.shape[1]):
        b = rhs[:, j]
        bnorm = float(np.sqrt(b @ b))
        if bnorm == 0.0:
            continue
        xc = x[:, j].copy()
        r = b - op(xc[:, None])[:, 0]
        p = r.copy()
        rr = float(r @ r)
        it = 0
        while math.sqrt(rr) > tol * bnorm and it < max_iter:
            ap = op(p[:, None])[:, 0]
            pap = float(p @ ap)
            if pap <= 0.0:
                breakdown = True
                break
            alpha = rr / pap
            xc += alpha * p
            r -= alpha * ap
            rr_new = float(r @ r)
            beta = rr_new / rr
            rr = rr_new
            p = r + beta * p
            it += 1
        max_used = max(max_used, it)
        x[:, j] = xc
    return x, breakdown, max_used


# ----------------------------------------------------------------------------------------------
# Dense host kernels (dense_kernels.cpp)
# ----------------------------------------------------------------------------------------------
def cholesky_lower(a):
    """A = L L^T or None when a pivot is <= 0 / non-finite (dense_kernels.cpp:11-28)."""
    n = a.shape[0]
    l = np.zeros((n, n))
    for j in range(n):
        d = a[j, j] - float(l[j, :j] @ l[j, :j])
        if not (d > 0.0) or not math.isfinite(d):
            return None
        ljj = math.sqrt(d)
        l[j, j] = ljj
        if j + 1 < n:
            l[j + 1:, j] = (a[j + 1:, j] - l[j + 1:, :j] @ l[j, :j]) / ljj
    return l


def jacobi_svd(a, max_sweeps=40):
    """One-sided cyclic Jacobi, conv 1e-15, sigma ascending (dense_kernels.cpp:30-113)."""
    a = np.array(a, dtype=np.float64, copy=True)
    m, k = a.shape
    if m < k:
        raise ContractViolation("jacobi_svd: requires rows >= cols")
    v = np.eye(k)
    rotated, sweep = True, 0
    while rotated and sweep < max_sweeps:
        rotated = False
        sweep += 1
        for p in range(k - 1):
            for q in range(p + 1, k):
                ap, aq = a[:, p], a[:, q]
                alpha = float(ap @ ap)
                beta = float(aq @ aq)
                gamma = float(ap @ aq)
                if alpha == 0.0 or beta == 0.0:
                    continue
                if abs(gamma) <= 1e-15 * math.sqrt(alpha * beta):
                    continue
                rotated = True
                zeta = (beta - alpha) / (2.0 * gamma)
                t = (1.0 if zeta >= 0.0 else -1.0) / (abs(zeta) + math.sqrt(1.0 + zeta * zeta))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = c * t
                a[:, p], a[:, q] = c * ap - s * aq, s * ap + c * aq
                vp, vq = v[:, p].copy(), v[:, q].copy()
                v[:, p], v[:, q] = c * vp - s * vq, s * vp + c * vq
    sig = np.sqrt(np.einsum("ij,ij->j", a, a))
    order = np.argsort(sig, kind="stable")
    sig = sig[order]
    inv = np.where(sig > 0.0, 1.0 / np.where(sig > 0, sig, 1.0), 0.0)
    u = a[:, order] * inv
    return u, sig, v[:, order], (not rotated), sweep


def spectral_norm(a):
    """Largest singular value via jacobi_svd (dense_kernels.cpp:115-123)."""
    if a.size == 0:
        return 0.0
    s = jacobi_svd(a if a.shape[0] >= a.shape[1] else a.T)[1]
    return float(s[-1])


# ----------------------------------------------------------------------------------------------
# Biorthogonalization (biorth.cpp)
# ----------------------------------------------------------------------------------------------
def _sign_or_plus(v):
    return -1.0 if v < 0.0 else 1.0


def gs_biorth(x, y, ip: InnerProduct, drop_tol, classical):
    """Column-sequential GS-Biorth with the drop rule and sign/sqrt|eta| scaling
    (biorth.cpp:19-69)."""
    if x.shape != y.shape:
        raise ContractViolation("biorth: X and Y must have equal shape")
    n, m = x.shape
    ps, qs, kept, dropped = [], [], [], []
    for l in range(m):
        pl, ql = x[:, l].copy(), y[:, l].copy()
        for pj, qj in zip(ps, qs):
            r = ip.dot(qj, x[:, l]) if classical else ip.dot(qj, pl)
            pl -= r * pj
            s = ip.dot(pj, y[:, l]) if classical else ip.dot(pj, ql)
            ql -= s * qj
        pnorm, qnorm = ip.norm(pl), ip.norm(ql)
        eta = ip.dot(pl, ql)
        if pnorm == 0.0 or qnorm == 0.0 or abs(eta) < drop_tol * pnorm * qnorm:
            dropped.append(l)
            continue
        scale = 1.0 / math.sqrt(abs(eta))
        ps.append(_sign_or_plus(eta) * pl * scale)
        qs.append(ql * scale)
        kept.append(l)
    p = np.stack(ps, axis=1) if ps else np.zeros((n, 0))
    q = np.stack(qs, axis=1) if qs else np.zeros((n, 0))
    return p, q, kept, dropped


def rebiorth_pass(p, q, ip: InnerProduct):
    """Second subtraction pass, no drop test (biorth.cpp:72-98)."""
    p, q = p.copy(), q.copy()
    for l in range(p.shape[1]):
        pl, ql = p[:, l].copy(), q[:, l].copy()
        for j in range(l):
            r = ip.dot(q[:, j], pl)
            pl -= r * p[:, j]
            s = ip.dot(p[:, j], ql)
            ql -= s * q[:, j]
        eta = ip.dot(pl, ql)
        if eta == 0.0:
            continue
        scale = 1.0 / math.sqrt(abs(eta))
        p[:, l] = _sign_or_plus(eta) * pl * scale
        q[:, l] = ql * scale
    return p, q


def biorth_residual(p, q, ip: InnerProduct):
    """||P^T Q - I||_2 (biorth.cpp:135-143)."""
    if p.shape[1] == 0:
        return 0.0
    g = block_inner(ip, p, q) - np.eye(p.shape[1])
    return spectral_norm(g)


def mgs_biorth(x, y, ip: InnerProduct = None, drop_tol=1e-12):
    """MGS-Biorth + conditional second pass when the loss exceeds 1e-10 (biorth.cpp:102-109)."""
    ip = ip or InnerProduct()
    p, q, kept, dropped = gs_biorth(x, y, ip, drop_tol, False)
    if p.shape[1] > 1 and biorth_residual(p, q, ip) > 1e-10:
        p, q = rebiorth_pass(p, q, ip)
    return p, q, kept, dropped


def cgs_biorth(x, y, ip: InnerProduct = None, drop_tol=1e-12):
    """Classical variant (biorth.cpp:111-114)."""
    return gs_biorth(x, y, ip or InnerProduct(), drop_tol, True)


def biorth_against(bases, x, y, ip: InnerProduct):
    """(I - sum P_k Q_k^T) X and (I - sum Q_k P_k^T) Y, sequential over bases
    (biorth.cpp:116-133)."""
    w, z = x.copy(), y.copy()
    for bp, bq in bases:
        if bp is None or bp.shape[1] == 0:
            continue
        w = block_axpy(bp, block_inner(ip, bq, w), w)
        z = block_axpy(bq, block_inner(ip, bp, z), z)
    return w, z


# ----------------------------------------------------------------------------------------------
# Projected LREP (projected_lrep.cpp)
# ----------------------------------------------------------------------------------------------
def finish_assembly(khat, mhat):
    """Symmetrize + two Cholesky or NullspaceLeak (projected_lrep.cpp:13-25)."""
    khat = 0.5 * (khat + khat.T)
    mhat = 0.5 * (mhat + mhat.T)
    lk = cholesky_lower(khat)
    if lk is None:
        raise NullspaceLeak("assemble_projected: U^T K U is not SPD")
    lm = cholesky_lower(mhat)
    if lm is None:
        raise NullspaceLeak("assemble_projected: V^T M V is not SPD")
    return khat, mhat, lk, lm


def solve_small_lrep(lk, lm, k):
    """W = L^T R, Jacobi SVD, Yhat = L Phi S^-1/2, Xhat = R Psi S^-1/2
    (projected_lrep.cpp:48-80)."""
    d = lk.shape[0]
    if k > d:
        raise ContractViolation("solve_small_lrep: k exceeds d")
    w = lk.T @ lm
    u, sig, v, _, _ = jacobi_svd(w)
    smax = sig[-1] if sig.size else 0.0
    if np.any(sig < 1e-14 * smax):
        raise DegenerateSpectrum("solve_small_lrep: singular value at round-off scale")
    inv = 1.0 / np.sqrt(sig[:k])
    return sig[:k].copy(), lm @ (v[:, :k] * inv), lk @ (u[:, :k] * inv)


# ----------------------------------------------------------------------------------------------
# Solver (bosp_solver.hpp / bosp_solver.cpp)
# ----------------------------------------------------------------------------------------------
@dataclass
class BospConfig:
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

    def effective_nb(self):  # bosp_solver.cpp:99-103
        if self.nb > 0:
            return min(self.nb, self.nev)
        return max(1, min((self.nev + 4) // 5, 150))

    def effective_moving(self):  # bosp_solver.cpp:105-108
        if self.moving is not None:
            return bool(self.moving)
        return self.nev > 3 * self.effective_nb()

    def validate(self):  # bosp_solver.cpp:110-115
        if self.nev == 0:
            raise ContractViolation("BospConfig: nev must be positive")
        if self.effective_nb() > self.nev:
            raise ContractViolation("BospConfig: nb exceeds nev")
        if self.s < 2:
            raise ContractViolation("BospConfig: s must be >= 2")
        if not self.tol > 0.0:
            raise ContractViolation("BospConfig: tol must be positive")


@dataclass
class SolverState:  # bosp_solver.hpp:53-69
    x: np.ndarray
    y: np.ndarray
    p: np.ndarray
    q: np.ndarray
    w: np.ndarray
    z: np.ndarray
    lambdas: list
    residuals: list
    frozen: int = 0
    nev_conv: int = 0
    locked: list = field(default_factory=list)          # [(P, Q)]
    locked_lambdas: list = field(default_factory=list)
    residual_history: list = field(default_factory=list)
    last_residual: list = field(default_factory=list)
    nevconv_history: list = field(default_factory=list)
    iter: int = 0
    leak_recovered: bool = False
    stats: dict = field(default_factory=lambda: dict(
        iterations=0, matvec_count=0, step3_matvecs=0, step3_vecprods=0, max_width_u=0,
        max_biorth_deviation=0.0, max_deflation_crossgram=0.0, final_biorth_deviation=0.0,
        nevconv_monotone=True, wall_seconds=0.0, repairs=0))


def _hcat(*blocks):
    blocks = [b for b in blocks if b is not None and b.shape[1] > 0]
    if not blocks:
        return None
    return np.concatenate(blocks, axis=1)


def _deflation_bases(st, ns):
    bases = []
    if ns is not None and ns[0].shape[1] > 0:
        bases.append(ns)
    bases += st.locked
    return bases


def _split(st, p, q, wx, wp, ww):
    st.x, st.p, st.w = p[:, :wx].copy(), p[:, wx:wx + wp].copy(), p[:, wx + wp:wx + wp + ww].copy()
    st.y, st.q, st.z = q[:, :wx].copy(), q[:, wx:wx + wp].copy(), q[:, wx + wp:wx + wp + ww].copy()


def initialize(K, M, ip, ns, cfg: BospConfig, n: int) -> SolverState:
    """Steps 1-2 (bosp_solver.cpp:117-177)."""
    cfg.validate()
    r = 0 if ns is None else ns[0].shape[1]
    budget = n - r
    if cfg.nev > budget:
        raise ContractViolation("bosp: nev exceeds the number of positive eigenvalues")
    nb = cfg.effective_nb()
    moving = cfg.effective_moving()
    wx = min(cfg.s * nb if moving else cfg.nev, budget)
    avail = budget - wx
    wp = min(nb, avail // 2)
    ww = min(nb, avail - wp)
    rng = MT19937_64(cfg.rng_seed)
    blocks = [fill_uniform(rng, n, w) for w in (wx, wp, ww, wx, wp, ww)]
    u = _hcat(blocks[0], blocks[1], blocks[2])
    v = _hcat(blocks[3], blocks[4], blocks[5])
    bases = [ns] if (ns is not None and ns[0].shape[1] > 0) else []
    u2, v2 = biorth_against(bases, u, v, ip)
    p, q, _, _ = mgs_biorth(u2, v2, ip)
    if p.shape[1] < wx + wp + ww:
        raise InitializationFailure("bosp: column drops during seeding")
    st = SolverState(None, None, None, None, None, None, [math.inf] * wx, [1.0] * wx)
    _split(st, p, q, wx, wp, ww)
    st.last_residual = [1.0] * cfg.nev
    return st


def _sample_invariants(st, ns, ip):
    """bosp_solver.cpp:63-76 (+ cross_gram_max :54-60)."""
    u = _hcat(st.x, st.p, st.w)
    v = _hcat(st.y, st.q, st.z)
    g = block_inner(ip, u, v) - np.eye(u.shape[1])
    dev = float(np.abs(g).max()) if g.size else 0.0
    st.stats["max_biorth_deviation"] = max(st.stats["max_biorth_deviation"], dev)
    cg = 0.0
    for bp, bq in _deflation_bases(st, ns):
        cg = max(cg, float(np.abs(block_inner(ip, bq, u)).max()), float(np.abs(block_inner(ip, bp, v)).max()))
    st.stats["max_deflation_crossgram"] = max(st.stats["max_deflation_crossgram"], cg)
    return dev


def _rebiorthogonalize_state(st, ns, ip):
    """bosp_solver.cpp:79-95."""
    st.stats["repairs"] += 1
    u = _hcat(st.x, st.p, st.w)
    v = _hcat(st.y, st.q, st.z)
    u2, v2 = biorth_against(_deflation_bases(st, ns), u, v, ip)
    p, q, _, dropped = mgs_biorth(u2, v2, ip)
    if dropped:
        raise NumericalAbort("bosp: rebiorthogonalization dropped columns")
    _split(st, p, q, st.x.shape[1], st.p.shape[1], st.w.shape[1])


def _ritz_step(st, K, M, u, v, k_extract):
    """Step 3 (bosp_solver.cpp:188-207)."""
    d = u.shape[1]
    ku, mv = K(u), M(v)
    st.stats["matvec_count"] += 2 * d
    st.stats["step3_matvecs"] += 2 * d
    st.stats["step3_vecprods"] += d * d + d
    khat, mhat, lk, lm = finish_assembly(u.T @ ku, v.T @ mv)
    lam, xh, yh = solve_small_lrep(lk, lm, k_extract)
    return dict(lam=lam, xhat=xh, yhat=yh, xt=u @ xh, yt=v @ yh, kxt=ku @ xh, myt=mv @ yh)


def iterate_once(st: SolverState, K, M, ip: InnerProduct, ns, cfg: BospConfig, n: int) -> bool:
    """Steps 3-7 (bosp_solver.cpp:211-435)."""
    nb = cfg.effective_nb()
    moving = cfg.effective_moving()
    r = 0 if ns is None else ns[0].shape[1]
    budget = n - r
    st.iter += 1
    st.stats["iterations"] += 1
    wxa = st.x.shape[1] - st.frozen
    u = _hcat(st.x[:, st.frozen:], st.p, st.w)
    v = _hcat(st.y[:, st.frozen:], st.q, st.z)
    st.stats["max_width_u"] = max(st.stats["max_width_u"], u.shape[1])
    try:
        sp_ = _ritz_step(st, K, M, u, v, wxa)
    except NullspaceLeak:
        if st.leak_recovered:
            raise NumericalAbort("bosp: projected blocks lost positive definiteness twice")
        st.leak_recovered = True
        _rebiorthogonalize_state(st, ns, ip)
        u = _hcat(st.x[:, st.frozen:], st.p, st.w)
        v = _hcat(st.y[:, st.frozen:], st.q, st.z)
        sp_ = _ritz_step(st, K, M, u, v, wxa)

    f = st.frozen
    st.x[:, f:] = sp_["xt"]
    st.y[:, f:] = sp_["yt"]
    for j in range(wxa):
        st.lambdas[f + j] = float(sp_["lam"][j])

    # Step 4 (:246-286)
    if ip.weighted:
        xt_b, yt_b = ip.weight(sp_["xt"]), ip.weight(sp_["yt"])
        st.stats["matvec_count"] += 2 * wxa
    else:
        xt_b, yt_b = sp_["xt"], sp_["yt"]
    lam = sp_["lam"]
    r1 = sp_["kxt"] - lam * yt_b
    r2 = sp_["myt"] - lam * xt_b
    num = np.einsum("ij,ij->j", r1, r1) + np.einsum("ij,ij->j", r2, r2)
    den = np.einsum("ij,ij->j", sp_["xt"], sp_["xt"]) + np.einsum("ij,ij->j", sp_["yt"], sp_["yt"])
    for j in range(wxa):
        st.residuals[f + j] = math.sqrt(num[j]) / ((1.0 + lam[j]) * math.sqrt(den[j]))
    base = len(st.locked_lambdas) + f
    prefix = 0
    while prefix < wxa and st.residuals[f + prefix] < cfg.tol:
        prefix += 1
    st.nev_conv = max(st.nev_conv, base + prefix)
    for j in range(wxa):
        if base + j >= cfg.nev:
            break
        st.last_residual[base + j] = st.residuals[f + j]
    st.residual_history.append(list(st.last_residual))
    if st.nevconv_history and st.nev_conv < st.nevconv_history[-1]:
        st.stats["nevconv_monotone"] = False
    st.nevconv_history.append(st.nev_conv)
    if st.nev_conv >= cfg.nev:
        return True

    # Step 5 (:288-327)
    d = u.shape[1]
    c0 = min(st.nev_conv - base, wxa)
    nb_eff = min(nb, wxa - c0)
    if wxa + 2 * nb_eff > budget:
        nb_eff = (budget - wxa) // 2
    ptil = qtil = np.zeros((n, 0))
    xh, yh = sp_["xhat"], sp_["yhat"]
    if nb_eff > 0:
        t1 = xh[:, c0:c0 + nb_eff].copy()
        t2 = yh[:, c0:c0 + nb_eff].copy()
        for j in range(nb_eff):
            t1[c0 + j, j] -= 1.0
            t2[c0 + j, j] -= 1.0
        phat = t1 - xh @ (yh.T @ t1)
        qhat = t2 - yh @ (xh.T @ t2)
        sp_p, sp_q, _, _ = mgs_biorth(phat, qhat, InnerProduct())
        if sp_p.shape[1] > 0:
            ptil, qtil = u @ sp_p, v @ sp_q

    # Step 6 (:329-388)
    wtil = ztil = np.zeros((n, 0))
    if nb_eff > 0:
        lam_b = lam[c0:c0 + nb_eff]
        rz_const = lam_b * xt_b[:, c0:c0 + nb_eff] - sp_["myt"][:, c0:c0 + nb_eff]
        rw_const = lam_b * yt_b[:, c0:c0 + nb_eff] - sp_["kxt"][:, c0:c0 + nb_eff]
        wgs = np.zeros((n, nb_eff))
        zgs = np.zeros((n, nb_eff))
        for sweep in range(cfg.ngs):
            rhs_z = rz_const.copy()
            if sweep > 0:
                bw = ip.weight(wgs) if ip.weighted else wgs
                rhs_z += lam_b * bw
            zgs, _, _ = cg_solve(M, rhs_z, np.zeros((n, nb_eff)), cfg.inner_cg_tol, cfg.inner_cg_max_iter)
            bz = ip.weight(zgs) if ip.weighted else zgs
            rhs_w = rw_const + lam_b * bz
            wgs, _, _ = cg_solve(K, rhs_w, np.zeros((n, nb_eff)), cfg.inner_cg_tol, cfg.inner_cg_max_iter)
        bases = _deflation_bases(st, ns) + [(st.x, st.y)]
        if ptil.shape[1] > 0:
            bases.append((ptil, qtil))
        wproj, zproj = biorth_against(bases, wgs, zgs, ip)
        wtil, ztil, _, _ = mgs_biorth(wproj, zproj, ip)

    # Step 7 (:390-427)
    st.p, st.q, st.w, st.z = ptil, qtil, wtil, ztil
    if moving:
        conv_window = st.nev_conv - len(st.locked_lambdas)
        if conv_window >= 2 * nb and st.x.shape[1] >= 2 * nb:
            st.locked.append((st.x[:, :2 * nb].copy(), st.y[:, :2 * nb].copy()))
            st.locked_lambdas += st.lambdas[:2 * nb]
            lam_rest = st.lambdas[2 * nb:]
            res_rest = st.residuals[2 * nb:]
            st.x = _hcat(st.x[:, 2 * nb:], st.p, st.w)
            st.y = _hcat(st.y[:, 2 * nb:], st.q, st.z)
            st.p = st.q = st.w = st.z = np.zeros((n, 0))
            st.lambdas = lam_rest + [math.inf] * (st.x.shape[1] - len(lam_rest))
            st.residuals = res_rest + [1.0] * (st.x.shape[1] - len(res_rest))
    else:
        if st.x.shape[1] > nb:
            milestone = nb * (st.nev_conv // nb)
            st.frozen = max(st.frozen, min(milestone, st.x.shape[1] - nb))

    if _sample_invariants(st, ns, ip) > 5e-11:
        _rebiorthogonalize_state(st, ns, ip)
    return False


@dataclass
class EigenResult:  # bosp_solver.hpp:71-81
    lambdas: np.ndarray
    x: np.ndarray
    y: np.ndarray
    iterations: int
    residuals: np.ndarray
    history: list
    nevconv_history: list
    converged: bool
    nev_converged: int
    stats: dict


def assemble_result(st, K, M, ip, cfg, converged, n) -> EigenResult:
    """bosp_solver.cpp:439-509."""
    have = min(cfg.nev, len(st.locked_lambdas) + st.x.shape[1])
    xs, ys, lams = [], [], []
    at = 0
    for bp, bq in st.locked:
        for j in range(bp.shape[1]):
            if at >= have:
                break
            xs.append(bp[:, j]); ys.append(bq[:, j]); lams.append(st.locked_lambdas[at]); at += 1
    j = 0
    while at < have and j < st.x.shape[1]:
        xs.append(st.x[:, j]); ys.append(st.y[:, j]); lams.append(st.lambdas[j]); at += 1; j += 1
    order = sorted(range(len(lams)), key=lambda i: lams[i])
    lam = np.array([lams[i] for i in order])
    x = np.stack([xs[i] for i in order], axis=1)
    y = np.stack([ys[i] for i in order], axis=1)
    kx, my = K(x), M(y)
    bx = ip.weight(x) if ip.weighted else x
    by = ip.weight(y) if ip.weighted else y
    r1 = kx - lam * by
    r2 = my - lam * bx
    num = np.einsum("ij,ij->j", r1, r1) + np.einsum("ij,ij->j", r2, r2)
    den = np.einsum("ij,ij->j", x, x) + np.einsum("ij,ij->j", y, y)
    res = np.sqrt(num) / ((1.0 + lam) * np.sqrt(den))
    stats = dict(st.stats)
    g = block_inner(ip, x, y) - np.eye(x.shape[1])
    stats["final_biorth_deviation"] = float(np.abs(g).max())
    return EigenResult(lam, x, y, st.iter, res, st.residual_history, st.nevconv_history,
                       converged, min(st.nev_conv, cfg.nev), stats)


def solve(K, M, ip: InnerProduct, cfg: BospConfig, ns, n: int) -> EigenResult:
    """bosp_solver.cpp:513-536 (the nullspace must be supplied)."""
    cfg.validate()
    t0 = time.perf_counter()
    st = initialize(K, M, ip, ns, cfg, n)
    converged = False
    while st.iter < cfg.max_outer_iter:
        if iterate_once(st, K, M, ip, ns, cfg, n):
            converged = True
            break
    res = assemble_result(st, K, M, ip, cfg, converged, n)
    res.stats["wall_seconds"] = time.perf_counter() - t0
    return res


def regression_coefficients(history, idx, tol):
    """log r_j = log alpha + beta log r_{j-1} (bosp_solver.cpp:538-580)."""
    r = [row[idx] for row in history if idx < len(row)]
    pts = []
    for j in range(1, len(r)):
        if not (r[j - 1] > 10.0 * tol) or not (r[j] > 10.0 * tol):
            continue
        if not (r[j - 1] > 0.0) or not (r[j] > 0.0):
            continue
        pts.append((math.log(r[j - 1]), math.log(r[j])))
    if len(pts) < 2:
        raise NotEnoughSamples("regression_coefficients: need at least 3 iterations")
    mx = sum(p[0] for p in pts) / len(pts)
    my = sum(p[1] for p in pts) / len(pts)
    sxx = sum((p[0] - mx) ** 2 for p in pts)
    sxy = sum((p[0] - mx) * (p[1] - my) for p in pts)
    if sxx < 1e-24:
        return math.exp(my), 0.0, True
    beta = sxy / sxx
    return math.exp(my - beta * mx), beta, False


# ----------------------------------------------------------------------------------------------
# Operator helpers
# ----------------------------------------------------------------------------------------------
def op_from_spec(spec):
    """("dense", A) | ("csr", (rowptr, colidx, vals)) | ("diag", d) -> apply(X)."""
    kind, payload = spec
    if kind == "dense":
        a = np.asarray(payload)
        return lambda x: a @ x
    if kind == "csr":
        import scipy.sparse as sp
        rp, ci, vv = payload
        a = sp.csr_matrix((vv, ci, rp), shape=(len(rp) - 1, len(rp) - 1))
        return lambda x: a @ x
    if kind == "diag":
        d = np.asarray(payload)[:, None]
        return lambda x: d * x
    if kind == "identity":
        return lambda x: x.copy()
    raise ValueError(kind)
