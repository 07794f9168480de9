"""Design of a per-step minimax sign-iteration schedule (Polar-Express style):
at step t the relative spectrum |mu| / ||A||_F lies in [l_t, u_t]; pick the odd
quintic p_t minimising max_{x in [l_t, u_t]} |1 - p_t(x)| (LP on a grid),
then [l_{t+1}, u_{t+1}] = p_t([l_t, u_t]). Eigenvalues below l_0 need no
accuracy (their projection error is <= l_0 ||A||_F). Prints the coefficients
and checks the composed map against the FP64 target.
    python tools/proto/sign_schedule_opt.py [l0] [safety]
"""
import sys

import numpy as np
from scipy.optimize import linprog


def minimax_quintic(l, u, cap=None):
    """min t s.t. 1 - t <= p(x) <= 1 + t on [l, u], written with t = 1 - s l
    and rows scaled by 1/x so that tiny l stays well conditioned:
    maximise s s.t. a + b x^2 + c x^4 >= s l / x  and  p(x) + s l <= 2."""
    xs = np.unique(np.concatenate([np.geomspace(l, u, 2000), np.linspace(l, u, 2000)]))
    lo = np.stack([-np.ones_like(xs), -xs ** 2, -xs ** 4, l / xs], 1)
    hi = np.stack([xs, xs ** 3, xs ** 5, np.full_like(xs, l)], 1)
    A_ub = np.vstack([lo, hi])
    b_ub = np.concatenate([np.zeros(len(xs)), 2.0 * np.ones(len(xs))])
    bounds = [(None, cap), (None, None), (None, None), (0, None)]
    r = linprog([0, 0, 0, -1], A_ub=A_ub, b_ub=b_ub, bounds=bounds, method="highs")
    a, b, c, sv = r.x
    return a, b, c, 1.0 - sv * l


def apply_range(p, l, u, a):
    xs = np.unique(np.concatenate([np.geomspace(l, u, 20001), np.linspace(l, u, 20001)]))
    ys = p(xs)
    lo = ys.min()
    if lo <= 100 * l * a * 1e-6 or lo < 1e-9:
        # the LP cannot resolve p near tiny l: p(x) = a x (1 + O(x^2)) there
        lo = min(lo, a * l) if lo > 0 else a * l
    return lo, ys.max()


def design(l0=1e-14, safety=1.0, tol=2e-16, max_steps=40):
    l, u = l0, 1.0
    steps = []
    for t in range(max_steps):
        a, b, c, err = minimax_quintic(l, u)
        p = lambda x, a=a, b=b, c=c: a * x + b * x ** 3 + c * x ** 5
        nl, nu = apply_range(p, l, u, a)
        steps.append((a, b, c, l, u, err))
        l, u = nl * safety, nu
        if err < tol:
            break
    return steps


def compose(steps, x):
    for a, b, c, *_ in steps:
        x = a * x + b * x ** 3 + c * x ** 5
    return x


if __name__ == "__main__":
    l0 = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-14
    safety = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    st = design(l0, safety)
    for i, (a, b, c, l, u, e) in enumerate(st):
        beta = b / (2 * c)
        gamma = a - b * b / (4 * c)
        xs = np.linspace(0, u, 200001)
        pm = np.abs(a * xs + b * xs ** 3 + c * xs ** 5).max()
        print(f"step {i:2d}: [{l:.3e}, {u:.6f}] a={a:.16g} b={b:.16g} c={c:.16g} err={e:.3e} "
              f"|p|max={pm:.3f} |U|<={max(abs(beta), abs(u * u + beta)):.3f} slope={a:.3f}")
    print(f"{len(st)} quintic steps = {3 * len(st)} GEMMs (+1 final)")
    xs = np.geomspace(1e-18, 1.0, 200001)
    f = compose(st, xs)
    print("max x|1-f(x)| over [1e-18, 1]:", np.max(xs * np.abs(1 - f)))
