"""Pins of the gradient-tally oracle (oracle/adjoint.py, Eq. 8, Alg. 1
line 12): the adjoint against central finite differences of the C oracle's
fp64 forward (an independent route: directional derivatives <lambda_0, e> for random e,
and single coordinates of every kind), the final-step case (lambda_T = m v_T), and the
bisection checkpointing against storing every state: identical tallies,
O(log T) resident states, O(T log T) forward steps."""
import math

import numpy as np
import pytest

from oracle import adjoint as adj
from paper_2207_04658_b200 import scenes


def z_of(sim, s0, T):
    s = np.asarray(s0, dtype=np.float64)
    for _ in range(T):
        s = adj.forward(sim, s)
    return adj.kinetic_energy(sim, s)


def lam0(sim, s0, T):
    s = [np.asarray(s0, dtype=np.float64)]
    for _ in range(T):
        s.append(adj.forward(sim, s[-1]))
    lam = adj.lambda_T(sim, s[T])
    for t in range(T - 1, -1, -1):
        lam = adj.adjoint_step(sim, s[t], lam)
    return lam


def make(material, **kw):
    return (scenes.adjoint_fluid if material == "fluid" else scenes.adjoint_elastic)(**kw)


@pytest.mark.parametrize("material", ["fluid", "elastic"])
@pytest.mark.parametrize("dim,T", [(2, 1), (2, 3), (3, 2)])
def test_adjoint_matches_finite_differences(material, dim, T):
    sim, s0 = make(material, dim=dim, side=6 if dim == 2 else 4, seed=dim + T)
    s0 = s0.astype(np.float64)
    lam = lam0(sim, s0, T)
    rng = np.random.default_rng(7)
    scale = np.ones(s0.shape[1])
    scale[:dim] = sim["dx"] * 1e-2  # positions: stay well inside a cell
    if material == "elastic":
        scale[2 * dim:2 * dim + dim * dim] = 1e-2  # the stiff F directions: small steps
    for trial in range(3):
        e = rng.normal(size=s0.shape) * scale
        eps = 1e-4
        fd = (z_of(sim, s0 + eps * e, T) - z_of(sim, s0 - eps * e, T)) / (2 * eps)
        an = float(np.sum(lam * e))
        assert abs(fd - an) <= 1e-6 * max(abs(fd), 1e-12) + 1e-9 * np.abs(lam * e).sum(), (trial, fd, an)


@pytest.mark.parametrize("material,dim", [("fluid", 2), ("elastic", 2), ("elastic", 3)])
def test_adjoint_single_coordinates_of_every_kind(material, dim):
    """One coordinate of each kind (x, v, J or F, C) of one particle: a dropped term in
    any branch of the adjoint fails here."""
    T = 2
    sim, s0 = make(material, dim=dim, side=5 if dim == 2 else 4, seed=3)
    s0 = s0.astype(np.float64)
    lam = lam0(sim, s0, T)
    p = 7
    for h in range(s0.shape[1]):
        e = np.zeros_like(s0)
        e[p, h] = sim["dx"] * 1e-2 if h < dim else (1e-2 if material == "elastic" and h < 2 * dim + dim * dim else 1.0)
        eps = 1e-4
        fd = (z_of(sim, s0 + eps * e, T) - z_of(sim, s0 - eps * e, T)) / (2 * eps)
        an = float(np.sum(lam * e))
        assert abs(fd - an) <= 1e-6 * max(abs(fd), abs(an)) + 1e-10, (h, fd, an)


def test_final_step_lambda_is_momentum():
    sim, s0 = scenes.adjoint_fluid(dim=2, side=4)
    z, g, lam = adj.backward_all(sim, s0, 0)
    d = 2
    m = sim["p_rho"] * sim["p_vol"]
    assert np.allclose(lam[:, d:2 * d], m * s0[:, d:2 * d].astype(np.float64))
    assert not lam[:, :d].any() and not lam[:, 2 * d:].any()
    assert np.allclose(g[d:2 * d], np.sum((m * s0[:, d:2 * d].astype(np.float64)) ** 2, 0))
    assert np.isclose(z, adj.kinetic_energy(sim, s0))


@pytest.mark.parametrize("T", [1, 2, 5, 8, 13])
def test_bisection_equals_store_all(T):
    sim, s0 = scenes.adjoint_fluid(dim=2, side=4, seed=T)
    z1, g1, l1 = adj.backward_all(sim, s0, T)
    st = {}
    z2, g2, l2 = adj.backward_bisection(sim, s0, T, stats=st)
    assert z1 == z2 and np.array_equal(g1, g2) and np.array_equal(l1, l2)
    assert st["max_resident"] <= math.ceil(math.log2(max(T, 1))) + 2, st
    assert st["forward_steps"] <= T + T * math.ceil(math.log2(max(T, 1))), st
