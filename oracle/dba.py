"""float64 CPU oracle of the DBA Gauss-Newton step — TEST INFRASTRUCTURE ONLY.

Restates ``/root/reference/SPEC.md:286-394`` (module ``dba``) on top of the
geometry restated in ``oracle/geometry.py``.  The reference has no dba code
(``pkg/src/flowsplat/__init__.py:8`` names the module; the file is absent), so
every convention the SPEC leaves open is fixed here and used identically by the
CUDA path:

  A1  left retraction  G <- exp(xi) o G                      (geometry.py:181-184)
  A2  relative pose    G_ij = G_j o G_i^-1                   (providers.py:327)
  A3  residual mask    weight * project-validity at the CURRENT state
                       (geometry.py:235-250)
  A4  damping          (S + lam*I) on the reduced pose(+intrinsics) system,
                       eta on the disparity diagonal C; lam0 = 1e-4; accept iff
                       E_trial <= E_cur, then lam = max(lam/10, 1e-8); reject ->
                       lam *= 10, stop (converged) once lam > 1e6.
                       A non-positive Cholesky pivot counts as a reject; if that
                       happens beyond lam_max -> SolverFailure.
  A5  mono gauge       pose(s) in ``fixed`` never move; when exactly one pose is
                       fixed and no disparity prior is used ("fix the mean
                       log-disparity of the first keyframe") every GN
                       step obeys the linearised, observation-weighted constraint
                       sum_p C_p dd_g,p / d_g,p = 0 on the gauge frame g (a hard
                       constraint eliminated with Sherman-Morrison: with c = C/d_g,
                       h = E C^-1 c = sum_p v_p / d_p, gamma = sum_p C_p / d_p^2,
                       rho = sum_p g_d,p / d_p the Schur complement gains
                       + h h^T / gamma, the rhs + h rho / gamma, and the
                       back-substitution becomes dd_p = r_p / C_p - kappa / d_p with
                       kappa = (rho - h . dx) / gamma).  Weighting by C keeps
                       unobserved pixels (C = eta) from absorbing the constraint.
                       The exact unweighted gauge is applied once at the end of the
                       call: s = exp(mean log d_g(input) - mean log d_g), d <- s*d,
                       and every pose moves by the similarity about camera g that
                       keeps G_g.
  A6  tangent clamp    per pose, ||xi_k||_2 <= 1, applied before back-substitution
                       
  A7  prior mask       explicit (N,H,W) mask input; C += alpha*m,
                       g_d += alpha*m*(d* - d)
  A8  edge order       input order is authoritative; CSR by source frame via a
                       stable sort; local Schur variables [i, j_e (CSR order), theta]
  A9  calib degeneracy ratio of largest/smallest Cholesky pivot of the
                       intrinsics block after pose elimination > CALIB_COND_MAX
  d_min = 1e-6 after every disparity update.

The normal equations use J = d(projection)/d(x) and g = J^T W r with
r = p* - projection, so the GN step solves (J^T W J) dx = g.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import geometry as G

CALIB_COND_MAX = 1e8


class OracleNumericalError(Exception):
    def __init__(self, msg, edge=-1):
        super().__init__(msg)
        self.edge = edge


class OracleSolverFailure(Exception):
    pass


class OracleCalibDegenerate(Exception):
    pass


@dataclass
class Options:
    iters: int = 4
    lam0: float = 1e-4
    lam_min: float = 1e-8
    lam_max: float = 1e6
    eta: float = 1e-4
    d_min: float = 1e-6
    tangent_max: float = 1.0
    optimize_intrinsics: bool = False
    alpha: float = 1e-3
    scale_gauge: bool | None = None  # None = auto (one fixed pose and no prior)
    # reduced-system solver: "cholesky" (LAPACK potrf, the reference path) or "lu" (LAPACK
    # getrf): an equally valid float64 ordering, used to measure the oracle's own
    # reproducibility floor on ill-conditioned problems (tests/golden/make_dba_golden.py)
    solver: str = "cholesky"
    # "reverse": the frame contributions to S, y and the energy are accumulated in reverse
    # frame order -- another valid float64 summation order (same use as ``solver``)
    order: str = "forward"


@dataclass
class Problem:
    """Edge list + per-edge (target, weight) as one (E,H,W,4) array [tu,tv,wu,wv]."""

    ii: np.ndarray
    jj: np.ndarray
    flow: np.ndarray
    fixed: np.ndarray  # (N,) bool
    prior: np.ndarray | None = None  # (N,H,W) disparity prior d*
    prior_mask: np.ndarray | None = None  # (N,H,W) {0,1}
    prior_weight: np.ndarray | None = None  # (N,) multiplier of alpha (Eq. 5 stage A: s^2)
    freeze_disparities: bool = False  # disparity block not updated (motion-only)

    @property
    def n_edges(self):
        return int(len(self.ii))


@dataclass
class State:
    poses: np.ndarray  # (N,7) float64
    disps: np.ndarray  # (N,H,W) float64
    intr: np.ndarray  # (4,) float64

    def copy(self):
        return State(self.poses.copy(), self.disps.copy(), self.intr.copy())


@dataclass
class Report:
    initial_energy: float
    final_energy: float
    iterations: int
    trials: int
    energy_trace: list = field(default_factory=list)
    converged: bool = False
    lam: float = 0.0


def csr_by_source(ii, n_frames):
    """Stable CSR of edges by source frame (A8).  Returns (offsets (N+1,), order (E,))."""
    ii = np.asarray(ii, dtype=np.int64)
    order = np.argsort(ii, kind="stable")
    counts = np.bincount(ii, minlength=n_frames)
    offs = np.zeros(n_frames + 1, dtype=np.int64)
    offs[1:] = np.cumsum(counts)
    return offs, order


# ----------------------------------------------------------------------------- per edge

def edge_terms(state: State, prob: Problem, e: int, calib: bool):
    """Residual, effective weight and Jacobians of one edge, non-homogeneous form.

    X_i = unproject(p, d_i)          (geometry.py:253-262)
    X_j = R_ij X_i + t_ij            (geometry.py:101-102, providers.py:327)
    pi  = project(X_j)               (geometry.py:235-250)
    J_j = J_pi(X_j) [I | -[X_j]x]                 (left perturbation of G_j)
    J_i = -J_pi(X_j) R_ij [I | -[X_i]x]           (left perturbation of G_i)
    J_d = J_pi(X_j) R_ij (-X_i / d)
    J_theta: d pi / d(fx,fy,cx,cy) through both unprojection and projection.
    Returns r (P,2), w (P,2), Ji, Jj (P,2,6), Jd (P,2), Jt (P,2,4) | None.
    """
    i, j = int(prob.ii[e]), int(prob.jj[e])
    fx, fy, cx, cy = state.intr
    _, h, w = state.disps.shape
    grid = G.pixel_grid(h, w).reshape(-1, 2)
    d = state.disps[i].reshape(-1)
    Xi = G.unproject(grid, d, state.intr)
    rel = G.relative_pose(state.poses, i, j)
    R = G.pose_R(rel)
    Xj = Xi @ R.T + rel[4:]
    pix, ok = G.project(Xj, state.intr, w, h)
    fl = prob.flow[e].reshape(-1, 4).astype(np.float64)
    r = fl[:, :2] - pix
    wt = fl[:, 2:4] * ok[:, None]

    Zs = np.where(ok, Xj[:, 2], 1.0)
    X, Y = Xj[:, 0], Xj[:, 1]
    P = len(d)
    Jp = np.zeros((P, 2, 3))
    Jp[:, 0, 0] = fx / Zs
    Jp[:, 0, 2] = -fx * X / Zs**2
    Jp[:, 1, 1] = fy / Zs
    Jp[:, 1, 2] = -fy * Y / Zs**2
    Jj = np.concatenate([Jp, np.cross(Xj[:, None, :], Jp)], axis=2)
    A = Jp @ R  # (P,2,3)
    Ji = -np.concatenate([A, np.cross(Xi[:, None, :], A)], axis=2)
    Jd = np.einsum("pck,pk->pc", A, -Xi / d[:, None])
    Jt = None
    if calib:
        xn = (grid[:, 0] - cx) / fx
        yn = (grid[:, 1] - cy) / fy
        dX = np.zeros((P, 3, 4))
        dX[:, 0, 0] = -xn / fx / d
        dX[:, 0, 2] = -1.0 / fx / d
        dX[:, 1, 1] = -yn / fy / d
        dX[:, 1, 3] = -1.0 / fy / d
        Jt = A @ dX
        Jt[:, 0, 0] += X / Zs
        Jt[:, 0, 2] += 1.0
        Jt[:, 1, 1] += Y / Zs
        Jt[:, 1, 3] += 1.0
    bad = ~ok
    r[bad] = 0.0
    for M in (Jj, Ji, Jd, Jt):
        if M is not None:
            M[bad] = 0.0
    return r, wt, Ji, Jj, Jd, Jt


def _wgram(wt, A, B):
    """sum_p sum_c w[p,c] A[p,c,:]^T B[p,c,:]."""
    a = (A * wt[:, :, None]).reshape(-1, A.shape[2])
    return a.T @ B.reshape(-1, B.shape[2])


def _wvec(wt, r, A):
    return ((wt * r)[:, :, None] * A).reshape(-1, A.shape[2]).sum(axis=0)


def _wpix(wt, Jd, A):
    """per-pixel coupling sum_c w Jd A  -> (P, k)."""
    return np.einsum("pc,pck->pk", wt * Jd, A)


# ----------------------------------------------------------------------------- system

@dataclass
class System:
    S: np.ndarray  # (6N+4, 6N+4) Schur-reduced system over ALL pose blocks + theta
    y: np.ndarray  # (6N+4,)
    energy: float
    edge_energy: np.ndarray  # (E,)
    edge_finite: np.ndarray  # (E,) bool
    C: np.ndarray  # (N,P)
    gd: np.ndarray  # (N,P)
    B: np.ndarray | None = None  # un-reduced pose block (for tests)


def _frame_terms(state, prob, opts, i, edges, calib, want_hessian):
    """Per-source-frame accumulation: C, g_d, coupling U (P, m) and the B blocks.

    U's columns are the local variables [i, j_e (CSR order), theta] (v-space)."""
    N = state.poses.shape[0]
    P = state.disps[i].size
    k = len(edges)
    m = 6 * (k + 1) + 4
    U = np.zeros((P, m))
    C = np.full(P, opts.eta)
    gd = np.zeros(P)
    energy = 0.0
    eng_e = {}
    fin_e = {}
    blocks = []  # (row_slice_global, col_slice_global, H) contributions
    grads = []
    th = slice(6 * N, 6 * N + 4)
    for a, e in enumerate(edges):
        j = int(prob.jj[e])
        r, wt, Ji, Jj, Jd, Jt = edge_terms(state, prob, e, calib)
        ee = float(np.sum(wt * r * r))
        eng_e[e] = ee
        energy += ee
        si, sj = slice(6 * i, 6 * i + 6), slice(6 * j, 6 * j + 6)
        if want_hessian:
            Hii = _wgram(wt, Ji, Ji)
            Hij = _wgram(wt, Ji, Jj)
            Hjj = _wgram(wt, Jj, Jj)
            blocks += [(si, si, Hii), (si, sj, Hij), (sj, si, Hij.T), (sj, sj, Hjj)]
            grads += [(si, _wvec(wt, r, Ji)), (sj, _wvec(wt, r, Jj))]
            if calib:
                Htt = _wgram(wt, Jt, Jt)
                Hti = _wgram(wt, Jt, Ji)
                Htj = _wgram(wt, Jt, Jj)
                blocks += [(th, th, Htt), (th, si, Hti), (si, th, Hti.T), (th, sj, Htj),
                           (sj, th, Htj.T)]
                grads += [(th, _wvec(wt, r, Jt))]
            fin_e[e] = bool(np.isfinite(Hjj).all() and np.isfinite(ee))
        U[:, 0:6] += _wpix(wt, Jd, Ji)
        U[:, 6 * (a + 1):6 * (a + 2)] += _wpix(wt, Jd, Jj)
        if calib:
            U[:, 6 * (k + 1):] += _wpix(wt, Jd, Jt)
        C += np.sum(wt * Jd * Jd, axis=1)
        gd += np.sum(wt * Jd * r, axis=1)
    if prob.prior is not None:
        dstar = prob.prior[i].reshape(-1).astype(np.float64)
        msk = prob.prior_mask[i].reshape(-1).astype(np.float64)
        dcur = state.disps[i].reshape(-1)
        al = prior_alpha(prob, opts, i)
        C += al * msk
        gd += al * msk * (dstar - dcur)
        energy += float(al * np.sum(msk * (dstar - dcur) ** 2))
    return U, C, gd, energy, eng_e, fin_e, blocks, grads


def prior_alpha(prob: Problem, opts: Options, i: int) -> float:
    """alpha of frame i's prior term (times the per-frame weight when given)."""
    if prob.prior_weight is None:
        return opts.alpha
    return opts.alpha * float(prob.prior_weight[i])


def _local_index(N, i, jlist):
    idx = list(range(6 * i, 6 * i + 6))
    for j in jlist:
        idx += list(range(6 * j, 6 * j + 6))
    idx += list(range(6 * N, 6 * N + 4))
    return np.array(idx)


def linearize(state: State, prob: Problem, opts: Options, frames=None,
              keep_B=False) -> System:
    """Schur-reduced normal equations at ``state``.

    For each source frame i (all frames when ``frames`` is None): accumulate the
    pose blocks B, the disparity diagonal C and the per-pixel pose/disparity
    couplings v_p (over the local variables [i, j_e..., theta]), then subtract
    the fill-in  sum_p v_p v_p^T / C_p  and  sum_p v_p g_d,p / C_p.
    ``frames`` restricts the sum to a frame subset (the sharded decomposition).
    """
    N = state.poses.shape[0]
    P = state.disps[0].size
    n_all = 6 * N + 4
    S = np.zeros((n_all, n_all))
    y = np.zeros(n_all)
    Bm = np.zeros((n_all, n_all)) if keep_B else None
    offs, order = csr_by_source(prob.ii, N)
    calib = opts.optimize_intrinsics
    Cs = np.zeros((N, P))
    gds = np.zeros((N, P))
    energy = 0.0
    E = prob.n_edges
    edge_energy = np.zeros(E)
    edge_finite = np.ones(E, dtype=bool)
    frame_list = range(N) if frames is None else frames
    if opts.order == "reverse":
        frame_list = list(frame_list)[::-1]
    g_frame = gauge_frame(prob, opts)
    gauge_terms = None
    for i in frame_list:
        edges = [int(x) for x in order[offs[i]:offs[i + 1]]]
        U, C, gd, en, eng_e, fin_e, blocks, grads = _frame_terms(
            state, prob, opts, i, edges, calib, True)
        energy += en
        for e, v in eng_e.items():
            edge_energy[e] = v
        for e, v in fin_e.items():
            edge_finite[e] = v
        for rs, cs, H in blocks:
            S[rs, cs] += H
            if keep_B:
                Bm[rs, cs] += H
        for rs, g in grads:
            y[rs] += g
        Cs[i] = C
        gds[i] = gd
        if (not edges and not calib) or prob.freeze_disparities:
            continue  # frozen disparities: no Schur fill-in, B and g stand alone
        idx = _local_index(N, i, [int(prob.jj[e]) for e in edges])
        Uc = U / C[:, None]
        S[np.ix_(idx, idx)] -= U.T @ Uc
        y[idx] -= Uc.T @ gd
        if i == g_frame:
            h, gam, rho = _gauge_terms(state, i, U, C, gd)
            S[np.ix_(idx, idx)] += np.outer(h, h) / gam
            y[idx] += h * rho / gam
            gauge_terms = (h, gam, rho)
    out = System(S, y, energy, edge_energy, edge_finite, Cs, gds, Bm)
    out.gauge = gauge_terms
    return out


def gauge_frame(prob: Problem, opts: Options):
    """Index of the gauge frame (first fixed pose) when the mono gauge is on, else -1."""
    if not use_scale_gauge(prob, opts):
        return -1
    return int(np.flatnonzero(prob.fixed)[0])


def _gauge_terms(state, i, U, C, gd):
    """A5 with c = C / d_i:  h = E C^-1 c = U^T (1/d),  gamma = sum C / d^2,
    rho = sum g_d / d."""
    inv_d = 1.0 / state.disps[i].reshape(-1)
    return U.T @ inv_d, float(np.sum(C * inv_d * inv_d)), float(np.sum(gd * inv_d))


def energy(state: State, prob: Problem, opts: Options | None = None) -> float:
    """Eq. 2 (+ Eq. 4 when a prior is given): sum_e sum_p w (.) r^2 over valid pixels
    (SPEC.md:304-312, 331-339)."""
    opts = opts or Options()
    N = state.poses.shape[0]
    tot = 0.0
    for e in range(prob.n_edges):
        r, wt, *_ = edge_terms(state, prob, e, False)
        tot += float(np.sum(wt * r * r))
    if prob.prior is not None:
        for i in range(N):
            dd = prob.prior[i].astype(np.float64) - state.disps[i]
            tot += float(prior_alpha(prob, opts, i) * np.sum(prob.prior_mask[i] * dd * dd))
    return tot


def free_index(fixed, calib):
    N = len(fixed)
    idx = []
    for k in range(N):
        if not fixed[k]:
            idx += list(range(6 * k, 6 * k + 6))
    if calib:
        idx += list(range(6 * N, 6 * N + 4))
    return np.array(idx, dtype=np.int64)


def reduced(sysm: System, prob: Problem, opts: Options):
    fi = free_index(prob.fixed, opts.optimize_intrinsics)
    return sysm.S[np.ix_(fi, fi)], sysm.y[fi], fi


def _chol_fast(A):
    """Cholesky via numpy (LAPACK) with the same failure semantics."""
    try:
        L = np.linalg.cholesky(A)
    except np.linalg.LinAlgError as exc:
        raise OracleSolverFailure(str(exc)) from None
    if not np.all(np.isfinite(L)):
        raise OracleSolverFailure("non-finite factor")
    return L


def solve_reduced(Sr, yr, lam, solver="cholesky"):
    import scipy.linalg
    A = Sr + lam * np.eye(Sr.shape[0])
    L = _chol_fast(A)
    if solver == "lu":
        return np.linalg.solve(A, yr), L
    z = scipy.linalg.solve_triangular(L, yr, lower=True)
    return scipy.linalg.solve_triangular(L, z, lower=True, trans=1), L


def clamp_tangents(dxi, tmax):
    """A6: scale each pose's 6-vector down to norm <= tmax."""
    out = dxi.copy()
    n = np.linalg.norm(out, axis=1)
    s = np.where(n > tmax, tmax / np.maximum(n, 1e-300), 1.0)
    return out * s[:, None]


def backsub_and_retract(state: State, prob: Problem, opts: Options, dxi_all, dth,
                        frames=None) -> State:
    """delta d_p = (g_d,p - v_p . delta_local) / C_p at the CURRENT state, then the
    retraction (A1), disparity floor d_min and theta += delta theta.
    ``dxi_all`` is (N,6) with zeros for fixed poses (already clamped)."""
    N = state.poses.shape[0]
    calib = opts.optimize_intrinsics
    offs, order = csr_by_source(prob.ii, N)
    new = state.copy()
    frame_list = range(N) if frames is None else frames
    g_frame = gauge_frame(prob, opts)
    for i in frame_list:
        if prob.freeze_disparities:
            continue
        edges = [int(x) for x in order[offs[i]:offs[i + 1]]]
        U, C, gd, *_ = _frame_terms(state, prob, opts, i, edges, calib, False)
        loc = [dxi_all[i]] + [dxi_all[int(prob.jj[e])] for e in edges]
        loc.append(dth if calib else np.zeros(4))
        dloc = np.concatenate(loc)
        vd = U @ dloc
        dd = (gd - vd) / C
        if i == g_frame and edges:
            h, gam, rho = _gauge_terms(state, i, U, C, gd)
            dd = dd - (rho - h @ dloc) / gam / state.disps[i].reshape(-1)
        new.disps[i] = np.maximum(state.disps[i] + dd.reshape(state.disps[i].shape),
                                  opts.d_min)
    for k in range(N):
        if not prob.fixed[k]:
            new.poses[k] = G.retract(state.poses[k], dxi_all[k])
    if calib:
        new.intr = state.intr + dth
    return new


def split_step(delta, fixed, calib):
    N = len(fixed)
    dxi = np.zeros((N, 6))
    o = 0
    for k in range(N):
        if not fixed[k]:
            dxi[k] = delta[o:o + 6]
            o += 6
    dth = delta[o:o + 4].copy() if calib else np.zeros(4)
    return dxi, dth


def use_scale_gauge(prob: Problem, opts: Options):
    if prob.freeze_disparities:
        return False
    if opts.scale_gauge is not None:
        return bool(opts.scale_gauge)
    return int(np.sum(prob.fixed)) == 1 and prob.prior is None


def apply_scale_gauge(state: State, prob: Problem, ref_disp_g, opts: Options):
    """A5: pin the mean log-disparity of the gauge frame g (first fixed pose)."""
    g = int(np.flatnonzero(prob.fixed)[0])
    s = float(np.exp(np.mean(np.log(ref_disp_g)) - np.mean(np.log(state.disps[g]))))
    out = state.copy()
    out.disps = np.maximum(state.disps * s, opts.d_min)
    Rg = G.pose_R(state.poses[g])
    tg = state.poses[g][4:]
    for k in range(state.poses.shape[0]):
        if k == g:
            continue
        Rk = G.pose_R(state.poses[k])
        c = Rk @ Rg.T @ tg
        out.poses[k][4:] = (state.poses[k][4:] - c) / s + c
    return out, s


def calib_condition(L, n_theta=4):
    """A9: ratio of the largest to smallest squared pivot of the theta block."""
    p = np.diag(L)[-n_theta:] ** 2
    return float(p.max() / max(p.min(), 1e-300))


def solve(state: State, prob: Problem, opts: Options | None = None, snapshot=None):
    """Damped Gauss-Newton with Schur elimination of disparities.

    ``snapshot(n, state, report)``, when given, is called after the n-th accepted
    iteration with the state an ``iters=n`` call would return (the A5 end-of-call gauge
    applied to a copy) -- the per-iteration fixtures in one run."""
    opts = opts or Options()
    calib = opts.optimize_intrinsics
    if not np.any(prob.fixed):
        raise ValueError("at least one pose must be fixed (gauge anchor)")
    cur = state.copy()
    ref_g = None
    gauge = use_scale_gauge(prob, opts)
    if gauge:
        g = int(np.flatnonzero(prob.fixed)[0])
        ref_g = state.disps[g].copy()
    sysm = linearize(cur, prob, opts)
    if not np.isfinite(sysm.energy) or not sysm.edge_finite.all():
        bad = int(np.flatnonzero(~sysm.edge_finite)[0]) if not sysm.edge_finite.all() else -1
        raise OracleNumericalError("non-finite residuals", bad)
    rep = Report(initial_energy=sysm.energy, final_energy=sysm.energy, iterations=0,
                 trials=0, lam=opts.lam0)
    lam = opts.lam0
    it = 0
    while it < opts.iters:
        Sr, yr, _ = reduced(sysm, prob, opts)
        try:
            delta, L = solve_reduced(Sr, yr, lam, opts.solver)
        except OracleSolverFailure:
            lam *= 10.0
            if lam > opts.lam_max:
                raise OracleSolverFailure("reduced system singular at maximum damping")
            continue
        if calib and calib_condition(L) > CALIB_COND_MAX:
            raise OracleCalibDegenerate("intrinsics block poorly conditioned")
        dxi, dth = split_step(delta, prob.fixed, calib)
        dxi = clamp_tangents(dxi, opts.tangent_max)
        trial = backsub_and_retract(cur, prob, opts, dxi, dth)
        tsys = linearize(trial, prob, opts)
        rep.trials += 1
        if not np.isfinite(tsys.energy) or not tsys.edge_finite.all():
            bad = int(np.flatnonzero(~tsys.edge_finite)[0]) if not tsys.edge_finite.all() else -1
            raise OracleNumericalError("non-finite residuals", bad)
        if tsys.energy <= sysm.energy:
            cur, sysm = trial, tsys
            lam = max(lam / 10.0, opts.lam_min)
            it += 1
            rep.energy_trace.append(sysm.energy)
            if snapshot is not None:
                snap = apply_scale_gauge(cur, prob, ref_g, opts)[0] if gauge else cur.copy()
                snapshot(it, snap, rep)
        else:
            lam *= 10.0
            if lam > opts.lam_max:
                rep.converged = True
                break
    rep.iterations = it
    rep.final_energy = sysm.energy
    rep.lam = lam
    if gauge:
        cur, _ = apply_scale_gauge(cur, prob, ref_g, opts)
    return cur, rep


# ----------------------------------------------------------------------------- dense check

def dense_joint_step(state: State, prob: Problem, opts: Options, lam: float):
    """Undamped-Schur reference: build the full joint system over
    [free pose tangents, theta, every disparity] and solve it densely.
    Only for tiny problems (AC3)."""
    N = state.poses.shape[0]
    _, h, w = state.disps.shape
    P = h * w
    calib = opts.optimize_intrinsics
    nv = 6 * N + 4 + N * P
    H = np.zeros((nv, nv))
    g = np.zeros(nv)
    dof = 6 * N + 4
    for e in range(prob.n_edges):
        i, j = int(prob.ii[e]), int(prob.jj[e])
        r, wt, Ji, Jj, Jd, Jt = edge_terms(state, prob, e, calib)
        J = np.zeros((P, 2, nv))
        J[:, :, 6 * i:6 * i + 6] = Ji
        J[:, :, 6 * j:6 * j + 6] = Jj
        if calib:
            J[:, :, 6 * N:6 * N + 4] = Jt
        for p in range(P):
            J[p, :, dof + i * P + p] = Jd[p]
        Jf = J.reshape(2 * P, nv)
        wf = wt.reshape(-1)
        H += Jf.T @ (Jf * wf[:, None])
        g += Jf.T @ (wf * r.reshape(-1))
    for i in range(N):
        for p in range(P):
            H[dof + i * P + p, dof + i * P + p] += opts.eta
    if prob.prior is not None:
        for i in range(N):
            m = prob.prior_mask[i].reshape(-1)
            dd = prob.prior[i].reshape(-1) - state.disps[i].reshape(-1)
            for p in range(P):
                H[dof + i * P + p, dof + i * P + p] += prior_alpha(prob, opts, i) * m[p]
                g[dof + i * P + p] += prior_alpha(prob, opts, i) * m[p] * dd[p]
    keep = list(free_index(prob.fixed, calib)) + list(range(dof, nv))
    keep = np.array(keep)
    Hk = H[np.ix_(keep, keep)]
    gk = g[keep]
    npose = len(free_index(prob.fixed, calib))
    Hk[np.arange(npose), np.arange(npose)] += lam
    gf = gauge_frame(prob, opts)
    if gf >= 0:  # A5: linearised gauge constraint as a KKT row
        a = np.zeros(len(keep))
        Cg = np.diag(H)[dof + gf * P:dof + (gf + 1) * P]
        a[npose + gf * P:npose + (gf + 1) * P] = Cg / state.disps[gf].reshape(-1)
        K = np.zeros((len(keep) + 1, len(keep) + 1))
        K[:-1, :-1] = Hk
        K[:-1, -1] = a
        K[-1, :-1] = a
        x = np.linalg.solve(K, np.concatenate([gk, [0.0]]))[:-1]
    else:
        x = np.linalg.solve(Hk, gk)
    return x[:npose], x[npose:].reshape(N, h, w)


def schur_step(state: State, prob: Problem, opts: Options, lam: float):
    """The same step through the Schur path (no clamp), for comparison with
    ``dense_joint_step``."""
    sysm = linearize(state, prob, opts)
    Sr, yr, _ = reduced(sysm, prob, opts)
    delta, _ = solve_reduced(Sr, yr, lam)
    dxi, dth = split_step(delta, prob.fixed, opts.optimize_intrinsics)
    N = state.poses.shape[0]
    calib = opts.optimize_intrinsics
    offs, order = csr_by_source(prob.ii, N)
    dd_all = np.zeros_like(state.disps)
    g_frame = gauge_frame(prob, opts)
    for i in range(N):
        edges = [int(x) for x in order[offs[i]:offs[i + 1]]]
        U, C, gd, *_ = _frame_terms(state, prob, opts, i, edges, calib, False)
        loc = [dxi[i]] + [dxi[int(prob.jj[e])] for e in edges]
        loc.append(dth if calib else np.zeros(4))
        dloc = np.concatenate(loc)
        dd = (gd - U @ dloc) / C
        if i == g_frame and edges:
            h, gam, rho = _gauge_terms(state, i, U, C, gd)
            dd = dd - (rho - h @ dloc) / gam / state.disps[i].reshape(-1)
        dd_all[i] = dd.reshape(dd_all[i].shape)
    return delta, dd_all
