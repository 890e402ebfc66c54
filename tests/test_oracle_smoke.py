"""Pins of the smoke oracle (oracle/smoke.py, DESIGN.md §12 readings S1-S8)
against what the mathematics fixes: exactness of trilinear sampling on linear fields,
the RK-3 order on a linear velocity field, central differences on linear fields, the
Jacobi fixed point of a quadratic, the Neumann/wall rules at the boundary, and the
advection-reflection step's special cases (dt = 0, a fluid at rest)."""
import numpy as np
import pytest

import oracle
from oracle import smoke as osm
from paper_2207_04658_b200 import scenes, schemes

RAW_U, RAW_P = schemes.smoke_raw(6), schemes.smoke_raw(2)


def grid_pos(res):
    return np.stack(np.meshgrid(*[np.arange(n) for n in res], indexing="ij"), -1).astype(np.float64)


def test_record_layout_S2():
    res = (6, 3, 4)
    f = np.random.default_rng(0).normal(size=res + (3,))
    rec = osm.to_records(f, 3)
    assert rec.shape == (3 * 3 * 4, 6)
    x, y, z = 3, 2, 1  # odd cell: record xr = 1, fields 3..5
    r = (1 * 3 + y) * 4 + z
    assert np.array_equal(rec[r, 3:], f[x, y, z]) and np.array_equal(rec[r, :3], f[2, y, z])
    assert np.array_equal(osm.from_records(rec, res, 3), f)


def test_sample_linear_exact_and_clamped_S3():
    res = (6, 5, 7)
    P = grid_pos(res)
    f = 0.3 * P[..., 0] - 1.2 * P[..., 1] + 0.7 * P[..., 2] + 2.0
    rng = np.random.default_rng(1)
    q = rng.uniform(0, 1, size=(200, 3)) * (np.array(res) - 1)
    lin = 0.3 * q[:, 0] - 1.2 * q[:, 1] + 0.7 * q[:, 2] + 2.0
    assert np.allclose(osm.sample(f, q), lin, rtol=0, atol=1e-12)
    # cell centres: the cell values (the top face too: i0 = n - 2, t = 1)
    assert np.allclose(osm.sample(f, P), f, atol=1e-12)
    # clamp to the domain
    out = q.copy()
    out[:, 0] = -3.5
    inside = q.copy()
    inside[:, 0] = 0.0
    assert np.allclose(osm.sample(f, out), osm.sample(f, inside), atol=1e-12)
    out[:, 0] = 99.0
    inside[:, 0] = res[0] - 1
    assert np.allclose(osm.sample(f, out), osm.sample(f, inside), atol=1e-12)
    # vector fields sample per component
    g = np.stack([f, 2 * f], -1)
    assert np.allclose(osm.sample(g, q)[:, 1], 2 * lin, atol=1e-11)


def test_backtrace_uniform_velocity_S4():
    res, dx, dt = (8, 6, 5), 0.1, 0.03
    u = np.broadcast_to(np.array([0.5, -0.25, 1.0]), res + (3,)).copy()
    xb = osm.backtrace(u, dt, dx)
    assert np.allclose(xb, grid_pos(res) - dt * u / dx, atol=1e-12)


def test_backtrace_is_third_order_on_a_rotation_S4():
    """u = w x (x - c), linear so trilinear sampling is exact: the departure point is
    exp(-dt A) x; Ralston's RK-3 has local error O(dt^4), so halving dt divides it by 16.
    (Swapping two weights, or Heun/midpoint coefficients, drops the order.)"""
    n, dx = 32, 1.0
    res = (n, n, n)
    P = grid_pos(res)
    c = (n - 1) / 2.0
    w = np.array([0.3, -0.2, 0.5])
    r = P - c
    u = np.cross(np.broadcast_to(w, r.shape), r) * dx  # world units: cells/s * dx
    A = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    sel = (np.abs(r) <= 4).all(-1)  # stay far from the clamp
    errs = []
    for dt in (0.2, 0.1):
        from scipy.linalg import expm
        exact = c + r[sel] @ expm(-dt * A).T
        errs.append(np.abs(osm.backtrace(u, dt, dx)[sel] - exact).max())
    assert errs[0] > 1e-9
    assert 12.0 < errs[0] / errs[1] < 20.0, errs


def test_divergence_linear_and_wall_S5():
    res, dx = (6, 5, 4), 0.25
    P = grid_pos(res) * dx
    u = np.stack([2.0 * P[..., 0], -0.5 * P[..., 1], 3.0 * P[..., 2]], -1)
    d = osm.divergence(u, dx)
    assert np.allclose(d[1:-1, 1:-1, 1:-1], 2.0 - 0.5 + 3.0, atol=1e-12)
    # a face cell sees u = 0 outside: x = 0 -> (u_x[1] - 0) / 2dx
    ux = u[..., 0]
    want = (ux[1, 2, 2] - 0.0) / (2 * dx) + (u[0, 3, 2, 1] - u[0, 1, 2, 1]) / (2 * dx) + \
        (u[0, 2, 3, 2] - u[0, 2, 1, 2]) / (2 * dx)
    assert np.isclose(d[0, 2, 2], want, atol=1e-12)


def test_jacobi_fixed_point_and_neumann_S6():
    res, dx = (7, 6, 5), 0.2
    P = grid_pos(res) * dx
    p = P[..., 0] ** 2 + P[..., 1] ** 2 - 0.5 * P[..., 2] ** 2  # 7-point Laplacian: 2 + 2 - 1 = 3
    out = osm.jacobi_sweep(p, np.full(res, 3.0), dx)
    assert np.allclose(out[1:-1, 1:-1, 1:-1], p[1:-1, 1:-1, 1:-1], atol=1e-12)
    # a constant pressure with no divergence is a fixed point everywhere (Neumann walls)
    c = np.full(res, 1.75)
    assert np.allclose(osm.jacobi_sweep(c, np.zeros(res), dx), c, atol=1e-15)
    # corner cell: 3 outside neighbours contribute p itself
    rng = np.random.default_rng(2)
    q = rng.normal(size=res)
    dv = rng.normal(size=res)
    want = (3 * q[0, 0, 0] + q[1, 0, 0] + q[0, 1, 0] + q[0, 0, 1] - dx * dx * dv[0, 0, 0]) / 6
    assert np.isclose(osm.jacobi_sweep(q, dv, dx)[0, 0, 0], want)


def test_jacobi_converges_to_the_neumann_poisson_solution_S6():
    """Many sweeps on a zero-mean right-hand side: the residual of the discrete Neumann
    Poisson problem sum_nb (p_nb - p) = dx^2 div goes to zero."""
    res, dx = (6, 5, 4), 1.0
    rng = np.random.default_rng(3)
    dv = rng.normal(size=res)
    dv -= dv.mean()
    p = np.zeros(res)
    for _ in range(3000):
        p = osm.jacobi_sweep(p, dv, dx)
    # independent residual: explicit neighbour loops
    r = np.zeros(res)
    for i in range(res[0]):
        for j in range(res[1]):
            for k in range(res[2]):
                s = 0.0
                for a, b, c in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
                    ii, jj, kk = i + a, j + b, k + c
                    inside = 0 <= ii < res[0] and 0 <= jj < res[1] and 0 <= kk < res[2]
                    s += (p[ii, jj, kk] if inside else p[i, j, k]) - p[i, j, k]
                r[i, j, k] = s - dx * dx * dv[i, j, k]
    assert np.abs(r).max() < 1e-6


def test_gradient_and_walls_S7():
    res, dx = (6, 5, 4), 0.5
    P = grid_pos(res) * dx
    p = 1.5 * P[..., 0] - 2.0 * P[..., 1] + 0.25 * P[..., 2]
    g = osm.gradient(p, dx)
    assert np.allclose(g[1:-1, 1:-1, 1:-1], [1.5, -2.0, 0.25], atol=1e-12)
    # Neumann at a wall: (p[1] - p[0]) / 2dx
    assert np.isclose(g[0, 2, 2, 0], (p[1, 2, 2] - p[0, 2, 2]) / (2 * dx))
    u = np.ones(res + (3,))
    w = osm.zero_walls(u)
    assert w[0, 2, 2, 0] == 0 and w[0, 2, 2, 1] == 1 and w[-1, 2, 2, 0] == 0
    assert w[2, 0, 2, 1] == 0 and w[2, -1, 2, 1] == 0 and w[2, 0, 2, 0] == 1
    assert w[2, 2, 0, 2] == 0 and w[2, 2, -1, 2] == 0
    assert w[1:-1, 1:-1, 1:-1].min() == 1


def test_store_raw_is_exact_and_fixed_is_within_a_quantum():
    res = (4, 3, 2)
    rng = np.random.default_rng(4)
    u = rng.normal(size=res + (3,)).astype(np.float32)
    _, back = osm.store(u.astype(np.float64), RAW_U, 0, 0, 3)
    assert np.array_equal(back.astype(np.float32), u)
    su = schemes.smoke_u()
    delta = su["fields"][0]["range"] * 2.0 ** -su["fields"][0]["frac_bits"]
    _, back = osm.store(0.5 * u.astype(np.float64) / np.abs(u).max(), su, 3, 7, 3)
    assert np.abs(back - 0.5 * u / np.abs(u).max()).max() < delta * (1 + 1e-6)


def test_fluid_at_rest_stays_at_rest_S8():
    """u = 0, p = 0, rho = 0: the step leaves u = p = 0 and sets rho = 1 in the source
    box only (any dropped/wrong-signed term would produce motion or density)."""
    params, _, _, _ = scenes.smoke(res=(8, 8, 6), amp=0.0, rho_blobs=0, jacobi_iters=4)
    res = params["res"]
    su, sp = schemes.smoke_u(), schemes.smoke_p()
    uw, _ = osm.store(np.zeros(res + (3,)), su, 0, 0, 3)
    pw, _ = osm.store(np.zeros(res + (1,)), sp, 0, 0, 1)
    un, pn, rho = osm.step((uw, pw, np.zeros(res, np.float32)), params, su, sp, 0, iters=4)
    assert not un.any() and not pn.any()
    lo, hi = params["source_lo"], params["source_hi"]
    box = np.zeros(res, bool)
    box[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = True
    assert (rho[box] == 1).all() and (rho[~box] == 0).all()


def test_buoyancy_enters_the_first_advection_S8():
    """Fluid at rest with rho = 1 in a box: u~_y = dt/2 b rho exactly (recorded value)."""
    params, _, _, _ = scenes.smoke(res=(8, 8, 6), amp=0.0, rho_blobs=0, jacobi_iters=2, buoyancy=3.0)
    res = params["res"]
    rho = np.zeros(res, np.float32)
    rho[2:5, 2:4, 1:3] = 1.0
    uw, _ = osm.store(np.zeros(res + (3,)), RAW_U, 0, 0, 3)
    pw, _ = osm.store(np.zeros(res + (1,)), RAW_P, 0, 0, 1)
    rec = []
    osm.step((uw, pw, rho), params, RAW_U, RAW_P, 0, iters=2, record=rec)
    kind, sub, ut = rec[0]
    assert kind == "u" and sub == 0
    assert np.allclose(ut[..., 1], 0.5 * params["dt"] * 3.0 * rho, atol=0)
    assert not ut[..., 0].any() and not ut[..., 2].any()


def test_zero_dt_keeps_density_S8():
    params, u, _, rho = scenes.smoke(res=(8, 6, 6), seed=5, jacobi_iters=3, dt=0.0)
    res = params["res"]
    uw, _ = osm.store(u.astype(np.float64), RAW_U, 0, 0, 3)
    pw, _ = osm.store(np.zeros(res + (1,)), RAW_P, 0, 0, 1)
    _, _, rho_n = osm.step((uw, pw, rho), params, RAW_U, RAW_P, 0, iters=3)
    lo, hi = params["source_lo"], params["source_hi"]
    want = rho.copy()
    want[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = 1.0
    assert np.array_equal(rho_n, want)


def test_reflection_uses_2uh_minus_ut_S8():
    """With dt = 0 both advections are the identity, so u' = 2 u_h - u~ and
    u_new = P(2 P(u) - u) (raw fp32 stores): checked against the composition of the
    pinned pieces."""
    params, u, _, rho = scenes.smoke(res=(8, 6, 6), seed=6, jacobi_iters=5, dt=0.0, buoyancy=0.0)
    res, dx = params["res"], params["dx"]
    uw, uq = osm.store(u.astype(np.float64), RAW_U, 0, 0, 3)
    pw, _ = osm.store(np.zeros(res + (1,)), RAW_P, 0, 0, 1)
    un, _, _ = osm.step((uw, pw, rho), params, RAW_U, RAW_P, 0, iters=5)
    got = osm.decode(un, RAW_U, res, 3)

    def P(v, p):
        d = osm.divergence(v, dx)
        for _ in range(5):
            p = np.float32(osm.jacobi_sweep(p, d, dx)).astype(np.float64)
        return np.float32(osm.zero_walls(v - osm.gradient(p, dx))).astype(np.float64), p

    uh, p1 = P(uq, np.zeros(res))
    want, _ = P(np.float32(2 * uh - uq).astype(np.float64), p1)
    assert np.allclose(got, want, rtol=1e-6, atol=1e-7)
