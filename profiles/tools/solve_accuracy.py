"""Accuracy of the banded block solves on the noisy C3 reduced system (numpy emulation).

The float64 oracle linearises the bench workload (C3, 0.5 px noise) at the state of golden
iteration n (0: the initial state), the reduced system S + lam I is solved by
  * LAPACK Cholesky (scipy),
  * block LDL^T with explicit pivot inverses and the update S_ac -= L_ab S_cb^T (round 1-2),
  * block Cholesky form of the updates, S_ac -= W_ab W_cb^T with W_ab = S_ab Li_b^T and the
    substitutions in LDL^T form (L_ab = W_ab Li_b, D_b^-1 = Li_b^T Li_b) -- dba_solve.cuh now,
and each step is compared with a 3x iteratively refined Cholesky solution (max-norm relative).

    python profiles/tools/solve_accuracy.py [n ...]       (CPU; ~15 s per state)
"""
import sys

import numpy as np
import scipy.linalg as sl

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests/golden")
from oracle import dba as O  # noqa: E402
from paper_2411_17660_b200 import scenes  # noqa: E402
import dba_codec  # noqa: E402

BW = 10


def system(n):
    g = np.load("/root/repo/tests/golden/dba_C3n.npz")
    wl = scenes.make_workload("C3", height=48, width=64, noise=0.5)
    if n == 0:
        P, D = wl.poses0.astype(np.float64), wl.disps0.astype(np.float64)
    else:
        refs = dba_codec.decode(wl.disps0, [g[f"dq_{k}"] for k in range(1, n + 1)])
        P, D = g[f"poses_{n}"], refs[n - 1]
    st = O.State(P.copy(), D.copy(), wl.intr0.astype(np.float64).copy())
    prob = O.Problem(ii=wl.ii, jj=wl.jj, flow=wl.flow, fixed=wl.fixed)
    opts = O.Options(iters=1)
    S, y = O.reduced(O.linearize(st, prob, opts), prob, opts)[:2]
    return S, y


def blk(A, a, b):
    return A[6 * a:6 * a + 6, 6 * b:6 * b + 6]


def ldl_explicit(A, y, nb):
    W = A.copy(); L = {}; Di = {}
    for b in range(nb):
        Di[b] = np.linalg.inv(blk(W, b, b))
        for a in range(b + 1, min(nb, b + BW + 1)):
            L[a, b] = blk(W, a, b) @ Di[b]
        for a in range(b + 1, min(nb, b + BW + 1)):
            for c in range(b + 1, a + 1):
                W[6 * a:6 * a + 6, 6 * c:6 * c + 6] -= L[a, b] @ blk(W, c, b).T
    return subst(y, nb, L, Di)


def chol_form(A, y, nb):
    W = A.copy(); L = {}; Di = {}; Wp = {}
    for b in range(nb):
        Li = sl.solve_triangular(np.linalg.cholesky(blk(W, b, b)), np.eye(6), lower=True)
        Di[b] = Li.T @ Li
        for a in range(b + 1, min(nb, b + BW + 1)):
            Wp[a] = blk(W, a, b) @ Li.T
            L[a, b] = Wp[a] @ Li
        for a in range(b + 1, min(nb, b + BW + 1)):
            for c in range(b + 1, a + 1):
                W[6 * a:6 * a + 6, 6 * c:6 * c + 6] -= Wp[a] @ Wp[c].T
    return subst(y, nb, L, Di)


def subst(y, nb, L, Di):
    z = y.copy()
    for b in range(nb):
        for a in range(b + 1, min(nb, b + BW + 1)):
            z[6 * a:6 * a + 6] -= L[a, b] @ z[6 * b:6 * b + 6]
    x = np.zeros_like(y)
    for b in range(nb - 1, -1, -1):
        xb = Di[b] @ z[6 * b:6 * b + 6]
        for a in range(b + 1, min(nb, b + BW + 1)):
            xb -= L[a, b].T @ x[6 * a:6 * a + 6]
        x[6 * b:6 * b + 6] = xb
    return x


def main():
    for n in [int(v) for v in sys.argv[1:]] or [0, 4]:
        S, y = system(n)
        A = S + 1e-4 * np.eye(S.shape[0])
        nb = S.shape[0] // 6
        c = sl.cho_factor(A)
        x = sl.cho_solve(c, y)
        for _ in range(3):
            x = x + sl.cho_solve(c, y - A @ x)
        err = lambda z: np.abs(z - x).max() / np.abs(x).max()  # noqa: E731
        print(f"state {n}: cond(S + 1e-4 I) {np.linalg.cond(A):.2e}   LAPACK Cholesky {err(sl.cho_solve(c, y)):.2e}"
              f"   block LDL^T explicit inverses {err(ldl_explicit(A, y, nb)):.2e}"
              f"   block Cholesky-form updates {err(chol_form(A, y, nb)):.2e}", flush=True)


if __name__ == "__main__":
    main()
