"""Pins for the oracle's MLS-MPM step (CPU only).

Closed forms (B-spline moments, affine reproduction, stress of a uniform scaling),
invariants (P2G mass/momentum conservation, rigid motion, free fall),
brute force (tiny 2D P2G over all nodes without stencil indexing) and a library
routine (numpy SVD for the polar decomposition).
"""
import numpy as np
import pytest

import oracle
from paper_2207_04658_b200 import scenes, schemes


def sim2d(res=16, E=0.0, g=(0.0, 0.0), bound=3, dt=1e-3, nu=0.2):
    return dict(dim=2, material="elastic", grid_res=(res, res, 1), dx=1.0 / res, dt=dt,
                gravity=(g[0], g[1], 0.0), p_rho=1.0, p_vol=(0.5 / res) ** 2, E=E, nu=nu, bound=bound)


def sim3d(res=16, E=0.0, g=(0.0, 0.0, 0.0), bound=3, dt=1e-3, material="elastic", nu=0.2):
    return dict(dim=3, material=material, grid_res=(res, res, res), dx=1.0 / res, dt=dt,
                gravity=tuple(g), p_rho=1.0, p_vol=(0.5 / res) ** 3, E=E, nu=nu, bound=bound)


def particle(d, x, v=None, F=None, C=None):
    v = np.zeros(d) if v is None else np.asarray(v, float)
    F = np.eye(d) if F is None else np.asarray(F, float)
    C = np.zeros((d, d)) if C is None else np.asarray(C, float)
    return np.concatenate([np.asarray(x, float), v, F.reshape(-1), C.reshape(-1)])


def node_positions(sim, origin, gsize):
    d = sim["dim"]
    axes = [(origin[a] + np.arange(gsize[a])) * sim["dx"] for a in range(d)]
    return np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)


# --------------------------------------------------------------- weights
def test_particle_on_node_masses_2d():
    """Particle on a node (fx = 1): w = (1/8, 3/4, 1/8); 2D masses 0.5625, 0.09375 x4,
    0.015625 x4 (times m_p)."""
    s = sim2d()
    st = particle(2, [5 * s["dx"], 7 * s["dx"]])[None]
    grid, origin, gsize, _ = oracle.p2g(s, st)
    m = grid[..., 0, 0] / (s["p_rho"] * s["p_vol"])
    assert tuple(origin[:2]) == (4, 6)
    w = np.array([0.125, 0.75, 0.125])
    np.testing.assert_allclose(m, np.outer(w, w), rtol=0, atol=1e-15)
    assert m[1, 1] == 0.5625 and m[0, 1] == 0.09375 and m[0, 0] == 0.015625


def test_particle_at_cell_centre_weights():
    """fx = 1/2: w = (1/2, 1/2, 0), the third node gets exactly zero weight."""
    s = sim2d()
    st = particle(2, [5.5 * s["dx"], 7.5 * s["dx"]])[None]
    grid, origin, gsize, _ = oracle.p2g(s, st)
    m = grid[..., 0, 0] / (s["p_rho"] * s["p_vol"])
    w = np.array([0.5, 0.5, 0.0])
    np.testing.assert_array_equal(m, np.outer(w, w))


@pytest.mark.parametrize("fx", [0.5, 0.7, 1.0, 1.3, 1.4999])
def test_bspline_moments(fx):
    """Sum w = 1, sum w (x_i - x_p) = 0, sum w (x_i - x_p)^2 = dx^2/4 per axis
    (quadratic B-spline, Hu et al. 2018) -- via the P2G mass distribution."""
    s = sim3d()
    dx = s["dx"]
    x = np.array([(6 + fx + 0.5) * dx, (5 + 0.5 + fx) * dx, (7 + 0.5 + 1.0) * dx])
    st = particle(3, x)[None]
    grid, origin, gsize, _ = oracle.p2g(s, st)
    m = grid[..., 0] / (s["p_rho"] * s["p_vol"])
    X = node_positions(s, origin, gsize)
    dpos = X - x
    assert abs(m.sum() - 1) < 1e-14
    for a in range(3):
        assert abs((m * dpos[..., a]).sum()) < 1e-15
        assert abs((m * dpos[..., a] ** 2).sum() / dx ** 2 - 0.25) < 1e-13


# --------------------------------------------------------------- conservation
def _random_state(d, n, res, rng, spread=0.05):
    x = rng.uniform(0.3, 0.7, (n, d))
    v = rng.normal(0, 1, (n, d))
    F = np.eye(d)[None] + spread * rng.normal(0, 1, (n, d, d))
    C = rng.normal(0, 5, (n, d, d))
    return np.concatenate([x, v, F.reshape(n, -1), C.reshape(n, -1)], axis=1)


@pytest.mark.parametrize("d", [2, 3])
def test_p2g_conserves_mass_and_momentum(d):
    """sum grid m = sum m_p and sum grid p = sum m_p v_p; the affine and stress
    terms cancel because sum_i w_ip (x_i - x_p) = 0.  fp64 to 1e-12 of the scale."""
    rng = np.random.default_rng(10 + d)
    s = sim2d(res=64, E=1e4) if d == 2 else sim3d(res=32, E=1e4)
    st = _random_state(d, 300, s["grid_res"][0], rng)
    grid, origin, gsize, oob = oracle.p2g(s, st)
    mp = s["p_rho"] * s["p_vol"]
    assert oob == 0
    assert abs(grid[..., 0].sum() - 300 * mp) <= 1e-12 * 300 * mp
    P = grid[..., 1:1 + d].reshape(-1, d).sum(axis=0)
    expect = mp * st[:, d:2 * d].sum(axis=0)
    scale = np.abs(grid[..., 1:1 + d]).sum()
    assert np.all(np.abs(P - expect) <= 1e-12 * scale)


def _bspline(r):
    r = abs(r)
    if r < 0.5:
        return 0.75 - r * r
    if r < 1.5:
        return 0.5 * (1.5 - r) ** 2
    return 0.0


def test_p2g_brute_force_tiny_2d():
    """Brute force: loop over ALL 64 nodes of an 8x8 grid with the B-spline kernel
    N((x_i - x_p)/dx) (zero outside its support), no stencil or base indexing."""
    rng = np.random.default_rng(7)
    s = sim2d(res=8, E=0.0)
    dx = s["dx"]
    mp = s["p_rho"] * s["p_vol"]
    for n in (1, 2, 3, 4):
        st = np.stack([particle(2, rng.uniform(2.2 * dx, 5.7 * dx, 2), rng.normal(0, 1, 2),
                                np.eye(2), rng.normal(0, 3, (2, 2))) for _ in range(n)])
        grid, origin, gsize, _ = oracle.p2g(s, st, origin=np.array([0, 0, 0]), gsize=np.array([8, 8, 1]))
        ref = np.zeros((8, 8, 3))
        for p in range(n):
            x, v, C = st[p, :2], st[p, 2:4], st[p, 8:12].reshape(2, 2)
            for i in range(8):
                for j in range(8):
                    xi = np.array([i, j]) * dx
                    w = _bspline((xi[0] - x[0]) / dx) * _bspline((xi[1] - x[1]) / dx)
                    ref[i, j, 0] += w * mp
                    ref[i, j, 1:] += w * (mp * v + mp * C @ (xi - x))
        np.testing.assert_allclose(grid[:, :, 0, :3], ref, rtol=0, atol=1e-15)


@pytest.mark.parametrize("d", [2, 3])
def test_stress_of_uniform_scaling(d):
    """F = s I: R = I, P F^T = [2 mu (s-1) s + lambda (s^d - 1) s^d] I (fixed corotated),
    so sum_i p_i,a (x_i - x_p)_a = -dt V_p 4/dx^2 k * dx^2/4 = -dt V_p k per axis."""
    E, nu, sc = 1000.0, 0.3, 1.07
    s = sim2d(E=E, nu=nu) if d == 2 else sim3d(E=E, nu=nu)
    x = np.full(d, 0.4317)
    st = particle(d, x, F=sc * np.eye(d))[None]
    grid, origin, gsize, _ = oracle.p2g(s, st)
    mu = E / (2 * (1 + nu))
    la = E * nu / ((1 + nu) * (1 - 2 * nu))
    k = 2 * mu * (sc - 1) * sc + la * (sc ** d - 1) * sc ** d
    X = node_positions(s, origin, gsize)
    g = grid if d == 3 else grid[:, :, 0, :]
    for a in range(d):
        moment = (g[..., 1 + a] * (X[..., a] - x[a])).sum()
        assert abs(moment - (-s["dt"] * s["p_vol"] * k)) <= 1e-12 * abs(s["dt"] * s["p_vol"] * k)


def test_rotation_has_zero_stress():
    """F = R (a rotation): F - R = 0, J = 1 => P F^T = 0; grid momentum = m v moments."""
    s = sim3d(E=5000.0)
    th = 0.3
    Rz = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1]])
    st = particle(3, [0.41, 0.52, 0.47], v=[0.3, -0.2, 0.1], F=Rz)[None]
    grid, origin, gsize, _ = oracle.p2g(s, st)
    mp = s["p_rho"] * s["p_vol"]
    np.testing.assert_allclose(grid[..., 1:], grid[..., :1] * np.array([0.3, -0.2, 0.1]), atol=1e-15 * mp)


# --------------------------------------------------------------- polar
@pytest.mark.parametrize("d", [2, 3])
def test_polar_matches_svd(d):
    """R = U V^T from numpy's SVD (library routine); orthogonal, det +1, R^T F symmetric."""
    rng = np.random.default_rng(20 + d)
    for _ in range(200):
        F = np.eye(d) + 0.3 * rng.normal(size=(d, d))
        if np.linalg.det(F) <= 0.05:
            continue
        R = oracle.polar(F)
        U, S, Vt = np.linalg.svd(F)
        Rs = U @ Vt
        np.testing.assert_allclose(R, Rs, atol=1e-11)
        np.testing.assert_allclose(R.T @ R, np.eye(d), atol=1e-12)
        assert abs(np.linalg.det(R) - 1) < 1e-12
        Sym = R.T @ F
        np.testing.assert_allclose(Sym, Sym.T, atol=1e-11)


def test_polar_of_rotation_is_itself():
    th = 1.1
    R0 = np.array([[1, 0, 0], [0, np.cos(th), -np.sin(th)], [0, np.sin(th), np.cos(th)]])
    np.testing.assert_allclose(oracle.polar(R0), R0, atol=1e-14)
    np.testing.assert_allclose(oracle.polar(2.5 * R0), R0, atol=1e-14)


# --------------------------------------------------------------- grid update
def test_boundary_separating_walls():
    """Reading Q13 (row a4): v_a = 0 if (i_a < bound and v_a < 0) or (i_a > n - bound
    and v_a > 0); other components and the interior untouched; v = p/m + dt g."""
    s = sim2d(res=16, g=(0.0, -10.0), dt=1e-3)
    grid = np.zeros((16, 16, 1, 4))
    grid[..., 0] = 2.0
    grid[..., 1] = 2.0 * -1.0  # v_x = -1
    grid[..., 2] = 2.0 * 0.5   # v_y = 0.5 before gravity
    out = oracle.grid_update(s, grid, np.array([0, 0, 0]), np.array([16, 16, 1]))
    vx, vy = out[:, :, 0, 1], out[:, :, 0, 2]
    assert np.all(vx[:3] == 0) and np.all(vx[3:] == -1.0)
    # vy > 0 after gravity: only the top wall (j > 16 - 3) zeroes it
    assert np.allclose(vy[:, :14], 0.5 - 1e-2) and np.all(vy[:, 14:] == 0)
    # empty nodes stay zero
    grid[..., 0] = 0.0
    out = oracle.grid_update(s, grid, np.array([0, 0, 0]), np.array([16, 16, 1]))
    assert np.all(out[..., 1:] == 0)


# --------------------------------------------------------------- G2P
@pytest.mark.parametrize("d", [2, 3])
def test_g2p_uniform_field(d):
    """A uniform grid velocity u gives v' = u and C' = 0 exactly (sum w = 1, sum w dpos = 0)."""
    rng = np.random.default_rng(30 + d)
    s = sim2d(res=32) if d == 2 else sim3d(res=32)
    st = _random_state(d, 50, 32, rng)
    origin, gsize = oracle.stencil_box(s, st)
    u = rng.normal(0, 1, 3)
    grid = np.zeros(tuple(gsize) + (4,))
    grid[..., 0] = 1.0
    grid[..., 1:1 + d] = u[:d]
    out = oracle.g2p(s, st, grid, origin, gsize)
    np.testing.assert_allclose(out[:, d:2 * d], np.broadcast_to(u[:d], (50, d)), atol=1e-14)
    np.testing.assert_allclose(out[:, -d * d:], 0.0, atol=1e-12)
    np.testing.assert_allclose(out[:, :d], st[:, :d] + s["dt"] * u[:d], atol=1e-15)


@pytest.mark.parametrize("d", [2, 3])
def test_g2p_affine_field(d):
    """v(x) = G x + b on the nodes gives v' = G x_p + b and C' = G (D_p = dx^2/4 I)."""
    rng = np.random.default_rng(40 + d)
    s = sim2d(res=32) if d == 2 else sim3d(res=32)
    st = _random_state(d, 50, 32, rng)
    origin, gsize = oracle.stencil_box(s, st)
    G = rng.normal(0, 2, (d, d))
    b = rng.normal(0, 1, d)
    X = node_positions(s, origin, gsize)
    grid = np.zeros(tuple(gsize) + (4,))
    V = X @ G.T + b
    if d == 2:
        grid[:, :, 0, 1:3] = V
    else:
        grid[..., 1:4] = V
    out = oracle.g2p(s, st, grid, origin, gsize)
    np.testing.assert_allclose(out[:, d:2 * d], st[:, :d] @ G.T + b, atol=1e-13)
    np.testing.assert_allclose(out[:, -d * d:].reshape(-1, d, d), np.broadcast_to(G, (50, d, d)), atol=1e-12)
    # F' = (I + dt C') F
    F = st[:, 2 * d:2 * d + d * d].reshape(-1, d, d)
    np.testing.assert_allclose(out[:, 2 * d:2 * d + d * d].reshape(-1, d, d),
                               (np.eye(d) + s["dt"] * G) @ F, atol=1e-13)


# --------------------------------------------------------------- full steps
def raw(dim, material="elastic"):
    return schemes.fp32(dim, material)


def _state_words(scheme, st):
    return oracle.encode_state(scheme, st.astype(np.float32))[0]


@pytest.mark.parametrize("d", [2, 3])
def test_rigid_translation(d):
    """F = I, C = 0, uniform v, no gravity, away from walls: v, C, F unchanged and
    x' = x + dt v."""
    rng = np.random.default_rng(50 + d)
    s = sim2d(res=32, E=300.0) if d == 2 else sim3d(res=32, E=300.0)
    n = 200
    x = rng.uniform(0.35, 0.65, (n, d))
    v = np.broadcast_to(np.array([0.7, -0.4, 0.2][:d]), (n, d))
    st = np.concatenate([x, v, np.broadcast_to(np.eye(d).reshape(-1), (n, d * d)), np.zeros((n, d * d))], 1)
    sch = raw(d)
    w = _state_words(sch, st)
    st32 = oracle.decode_state(sch, w).astype(np.float64)
    pre, _, _ = oracle.step(s, sch, w, 1)
    np.testing.assert_allclose(pre[:, d:2 * d], st32[:, d:2 * d], atol=1e-12)
    np.testing.assert_allclose(pre[:, :d], st32[:, :d] + s["dt"] * st32[:, d:2 * d], atol=1e-13)
    np.testing.assert_allclose(pre[:, 2 * d:2 * d + d * d], st32[:, 2 * d:2 * d + d * d], atol=1e-12)
    np.testing.assert_allclose(pre[:, -d * d:], 0.0, atol=1e-9)


def test_rigid_rotation_2d():
    """E = 0, v = w x (x - xc), C = skew(w): the affine field is reproduced exactly,
    so v and C are unchanged (APIC/MLS-MPM preserves affine motion)."""
    rng = np.random.default_rng(60)
    s = sim2d(res=32, E=0.0)
    n = 300
    x = rng.uniform(0.35, 0.65, (n, 2))
    om, xc = 2.0, np.array([0.5, 0.5])
    v = om * np.stack([-(x[:, 1] - xc[1]), x[:, 0] - xc[0]], 1)
    C = np.broadcast_to(np.array([0.0, -om, om, 0.0]), (n, 4))
    st = np.concatenate([x, v, np.broadcast_to(np.eye(2).reshape(-1), (n, 4)), C], 1)
    pre, _, _ = oracle.step(s, raw(2), _state_words(raw(2), st), 1)
    st32 = oracle.decode_state(raw(2), _state_words(raw(2), st)).astype(np.float64)
    np.testing.assert_allclose(pre[:, 2:4], st32[:, 2:4], atol=1e-6)
    np.testing.assert_allclose(pre[:, 8:12], st32[:, 8:12], atol=1e-5)


def test_free_fall_and_rest():
    """with E = 0 and no walls, v_T = v_0 + T dt g; a single particle at
    rest with no gravity is a fixed point."""
    s = sim3d(res=32, E=0.0, g=(0.0, -9.8, 0.0), bound=0, dt=1e-3)
    rng = np.random.default_rng(70)
    n = 100
    x = rng.uniform(0.4, 0.6, (n, 3))
    st = np.concatenate([x, np.zeros((n, 3)), np.broadcast_to(np.eye(3).reshape(-1), (n, 9)),
                         np.zeros((n, 9))], 1)
    w = _state_words(raw(3), st)
    for t in range(1, 6):
        pre, w, _ = oracle.step(s, raw(3), w, t)
    np.testing.assert_allclose(pre[:, 4], -9.8 * 5 * 1e-3, rtol=1e-5)
    s0 = sim3d(res=32, E=100.0)
    st1 = particle(3, [0.51, 0.47, 0.53])[None]
    w1 = _state_words(raw(3), st1)
    pre, w2, _ = oracle.step(s0, raw(3), w1, 1)
    assert np.array_equal(w1, w2)


def test_fluid_at_rest_is_a_fixed_point():
    """Fluid (reading Q15) at rest with J = 1, C = 0 and no gravity: nothing moves (the
    J = 1 special case of the closed forms below)."""
    s = sim3d(res=32, E=50.0, material="fluid")
    rng = np.random.default_rng(80)
    n = 100
    st = np.concatenate([rng.uniform(0.4, 0.6, (n, 3)), np.zeros((n, 3)), np.ones((n, 1)), np.zeros((n, 9))], 1)
    sch = schemes.fp32(3, "fluid")
    w = _state_words(sch, st)
    pre, w2, _ = oracle.step(s, sch, w, 1)
    np.testing.assert_array_equal(w, w2)


def fluid_particle(x, v=(0, 0, 0), J=1.0, C=None):
    C = np.zeros((3, 3)) if C is None else np.asarray(C, float)
    return np.concatenate([np.asarray(x, float), np.asarray(v, float), [J], C.reshape(-1)])


@pytest.mark.parametrize("J", [0.9, 0.97, 1.06])
def test_fluid_stress_first_moment_closed_form(J):
    """P2G of the J-fluid stress (reading Q15: P F^T = E (J - 1) I, affine
    A = -dt V_p 4/dx^2 P F^T): with v = 0 and C = 0 the node momenta are p_i = w_i A (x_i -
    x_p), so sum_i p_i = 0 and sum_i p_i (x) (x_i - x_p) = A dx^2/4 = -dt V_p E (J - 1) I
    (B-spline second moment 1/4 per axis).  A sign or scale error in E (J - 1), or an extra
    J factor, changes the moment."""
    E, dt = 40.0, 2e-4
    s = sim3d(res=32, E=E, dt=dt, material="fluid")
    xp = np.array([0.4731, 0.5212, 0.4968])
    grid, origin, gsize, _ = oracle.p2g(s, fluid_particle(xp, J=J)[None])
    X = node_positions(s, origin, gsize) - xp
    p = grid[..., 1:4]
    mom = np.einsum("xyza,xyzb->ab", p, X)
    expect = -dt * s["p_vol"] * E * (J - 1.0) * np.eye(3)
    np.testing.assert_allclose(mom, expect, rtol=1e-12, atol=1e-12 * abs(expect[0, 0]))
    np.testing.assert_allclose(p.sum(axis=(0, 1, 2)), 0.0, atol=1e-12 * abs(expect[0, 0]) / s["dx"])
    assert np.isclose(grid[..., 0].sum(), s["p_rho"] * s["p_vol"], rtol=1e-14)


@pytest.mark.parametrize("J", [0.95, 1.02])
def test_fluid_J_update_affine_field(J):
    """G2P of the J-fluid (reading Q11/Q15): an affine grid velocity v(x) = G x + b
    gives C' = G (affine reproduction) and J' = J (1 + dt tr C') = J (1 + dt tr G); a
    dropped J, a flipped sign or tr over the wrong entries fails."""
    s = sim3d(res=32, dt=1e-3, material="fluid")
    rng = np.random.default_rng(81)
    G = rng.normal(0, 3.0, (3, 3))
    b = rng.normal(0, 1.0, 3)
    st = fluid_particle([0.4812, 0.5377, 0.5091], J=J)[None]
    origin, gsize = oracle.stencil_box(s, st)
    Xn = node_positions(s, origin, gsize)
    grid = np.zeros(tuple(int(g) for g in gsize[:3]) + (4,))
    grid[..., 0] = 1.0
    grid[..., 1:4] = Xn @ G.T + b
    out = oracle.g2p(s, st, grid, origin, gsize)[0]
    np.testing.assert_allclose(out[7:16].reshape(3, 3), G, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(out[3:6], G @ st[0, :3] + b, rtol=1e-12, atol=1e-12)
    assert np.isclose(out[6], J * (1.0 + s["dt"] * np.trace(G)), rtol=1e-13, atol=0)


@pytest.mark.parametrize("J", [0.9, 1.05])
def test_fluid_single_particle_step_closed_form(J):
    """One whole fluid step of a lone particle (no gravity, away from walls): P2G gives
    p_i = w_i A (x_i - x_p), m_i = w_i m_p, so the grid velocity is the affine field
    (A / m_p)(x_i - x_p) and G2P returns v' = 0, C' = A / m_p and
    J' = J (1 + dt tr A / m_p) = J (1 - 12 dt^2 E (J - 1) / (rho dx^2)):
    a compressed particle (J < 1) expands.  Exercises the stress and the J update together."""
    E, dt = 30.0, 1e-4
    s = sim3d(res=32, E=E, dt=dt, material="fluid")
    st = fluid_particle([0.4903, 0.5066, 0.5127], J=J)[None]
    sch = schemes.fp32(3, "fluid")
    w = _state_words(sch, st)
    pre, _, _ = oracle.step(s, sch, w, 1)
    Jf = float(np.float32(J))
    A = -dt * s["p_vol"] * 4.0 / s["dx"] ** 2 * E * (Jf - 1.0)
    mp = s["p_rho"] * s["p_vol"]
    np.testing.assert_allclose(pre[0, 3:6], 0.0, atol=1e-12)
    np.testing.assert_allclose(pre[0, 7:16].reshape(3, 3), A / mp * np.eye(3), rtol=1e-9, atol=1e-9 * abs(A / mp))
    Jexp = Jf * (1.0 - 12.0 * dt * dt * E * (Jf - 1.0) / (s["p_rho"] * s["dx"] ** 2))
    assert np.isclose(pre[0, 6], Jexp, rtol=1e-12, atol=0)
    assert (pre[0, 6] > Jf) == (Jf < 1.0)


# --------------------------------------------------------------- consistency
def test_f32_matches_f64_on_c1():
    sc = scenes.c1()
    sch = schemes.x16()
    w, _ = oracle.encode_state(sch, sc.state())
    p64, w64, _ = oracle.step(sc.sim, sch, w, 1, "f64")
    p32, w32, _ = oracle.step(sc.sim, sch, w, 1, "f32")
    scale = np.maximum(np.abs(p64), 1e-3)
    assert np.max(np.abs(p32 - p64) / scale) < 1e-4


def test_sampled_step_equals_full_step():
    sc = scenes.small_elastic_3d()
    sch = schemes.e01()
    w, _ = oracle.encode_state(sch, sc.state())
    w1, _ = oracle.run(sc.sim, sch, w, 1, 3)
    pre, wout, _ = oracle.step(sc.sim, sch, w1, 4)
    sample = np.array([0, 7, 100, 1999, sc.n_particles - 1], dtype=np.uint64)
    spre, swords = oracle.step_sampled(sc.sim, sch, w1, 4, sample)
    np.testing.assert_allclose(spre, pre[sample.astype(np.int64)], rtol=1e-13, atol=1e-13)
    assert np.array_equal(swords, wout[sample.astype(np.int64)])


def test_dither_keys_are_content_keyed():
    """Reading Q5: permuting particles permutes the output words identically."""
    sc = scenes.small_elastic_3d()
    sch = schemes.e01()
    w, _ = oracle.encode_state(sch, sc.state())
    perm = np.random.default_rng(0).permutation(w.shape[0])
    _, a, ca = oracle.step(sc.sim, sch, w, 1)
    _, b, cb = oracle.step(sc.sim, sch, w[perm], 1)
    assert np.array_equal(a[perm], b)
    # (the up/down counters may differ: a value ~1e-17 either side of a grid point
    #  rounds to the same code via "down" or "up" depending on fp64 sum order)


@pytest.mark.parametrize("mk", [scenes.small_elastic_3d, scenes.small_fluid_3d])
def test_openmp_oracle_equals_serial(mk):
    """The OpenMP oracle (SURVEY §8(d) M7 ii) runs the same arithmetic with a different
    P2G summation order (4-cell x slabs): fp64 results agree to round-off, the words are
    identical but for rounding-boundary ties, and the result does not depend on the
    thread count."""
    sc = mk()
    sch = schemes.f2() if sc.material == "fluid" else schemes.e01()
    w, _ = oracle.encode_state(sch, sc.state())
    w, _ = oracle.run(sc.sim, sch, w, 1, 3)
    p1, w1, c1 = oracle.step(sc.sim, sch, w, 4)
    p8, w8, c8 = oracle.step(sc.sim, sch, w, 4, threads=8)
    p2, w2, c2 = oracle.step(sc.sim, sch, w, 4, threads=2)
    scale = np.maximum(np.abs(p1).max(axis=0), 1e-12)
    assert np.max(np.abs(p8 - p1) / scale) < 1e-8  # (C is a cancelling sum: round-off ~ 4/dx |v| eps)
    assert np.mean(np.any(w8 != w1, axis=1)) < 1e-3
    assert np.array_equal(p8, p2) and np.array_equal(w8, w2) and np.array_equal(c8, c2)
    wr, _ = oracle.run(sc.sim, sch, w, 4, 3, threads=4)
    wr2, _ = oracle.run(sc.sim, sch, w, 4, 3, threads=3)
    assert np.array_equal(wr, wr2)
