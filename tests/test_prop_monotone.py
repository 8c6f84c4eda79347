"""Property: within a multi-turn class (queue, tau) the IMPLEMENTED priority
P = ((alpha * w) * 0.5 erfc(z / sqrt2)) / dt, z = (ln dt - mu) / sigma, is non-increasing in dt
(SURVEY 8(a) a4).  The select's candidate shortcut for the multi-turn classes (their k'
oldest blocks are their k' lowest-priority blocks) rests on it, and its exactness check adds
a 2^-30 relative margin on top.  Checked on dense log grids over [1e-4, 1e7] s, on chains of
ulp-adjacent dt around points across the range (where fdlibm rounding could break it), and
on the clamp / cut-off edges, for the default parameters, C5 grid points and extreme
(mu, sigma) including the sigma floor 0.1."""
import math

import numpy as np
import pytest

import oracle
from paper_2605_18825_b200 import configs as C


def param_sets():
    out = [C.DEFAULT_PARAMS, C.c5_point_params(0), C.c5_point_params(29)]
    for mu, sg in ((0.0, 0.1), (4.82, 1.25), (2.28, 1.34), (12.0, 0.1), (-3.0, 3.0), (8.0, 0.35)):
        p = dict(C.DEFAULT_PARAMS)
        p["mu"], p["sigma"] = [mu, mu], [sg, sg]
        p["alpha"], p["w"] = [1.7, 0.3, 1.0], [4.13, 2.0, 1.8, 1.86, 0.77]
        out.append(p)
    return out


def dt_grid(seed=0):
    rng = np.random.default_rng(seed)
    g = list(np.logspace(-4, 7, 6000))
    for c in list(np.logspace(-3, 6.5, 40)) + [1e-3, math.e, 63.43, 110.6]:
        x = float(c)
        for _ in range(60):                 # ulp-adjacent chain
            g.append(x)
            x = math.nextafter(x, math.inf)
    g += list(rng.uniform(1e-3, 5e3, 2000))
    return np.unique(np.array(g, np.float64))


@pytest.mark.parametrize("pi", range(9))
def test_multiturn_priority_nonincreasing_in_dt(pi):
    p = param_sets()[pi]
    g = dt_grid(pi)
    for q in (1, 2):
        for tau in range(4):
            P = np.array([oracle.priority(p, q, tau, float(x)) for x in g])
            bad = np.nonzero(P[1:] > P[:-1])[0]
            assert len(bad) == 0, (pi, q, tau, g[bad[:3]], P[bad[:3]], P[bad[:3] + 1])
            assert np.all(P >= 0.0)


def test_priority_edges():
    p = dict(C.DEFAULT_PARAMS)
    # dt <= eps is clamped to eps (A7): all equal
    v = {oracle.priority(p, 1, 1, x) for x in (0.0, 1e-9, 1e-3)}
    assert len(v) == 1
    # beyond the survival cut-off (z > 30) the priority is exactly 0 (A36)
    p["mu"], p["sigma"] = [0.0, 0.0], [0.1, 0.1]
    assert oracle.priority(p, 1, 1, math.exp(3.0000001)) == 0.0
    assert oracle.priority(p, 1, 1, math.exp(2.99)) > 0.0
