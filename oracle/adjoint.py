"""Oracle of the gradient tallies g_h (Algorithm 1 line 12, Eq. 8,
P:337-339; Section "Gradient Computation") -- numpy fp64.

TEST INFRASTRUCTURE ONLY (same rule as the rest of oracle/).  Shares no code with
paper_2207_04658_b200/csrc/adjoint.cu.  The forward step is the C oracle's fp64
p2g -> grid_update -> g2p (oracle/mpm_impl.h); this file adds its adjoint.

Scope: both materials, 2D and 3D -- the J-fluid (reading Q15:
P F^T = E (J-1) I) and the fixed-corotated elastic (P F^T = 2 mu (F - R) F^T +
lambda (J-1) J I) with the polar decomposition's derivative: from F = R S,
skew(R^T dF) = (Omega S + S Omega)/2 with Omega = R^T dR, so (3D) the axial vector of
Omega is (tr(S) I - S)^{-1} axial(R^T dF - dF^T R) and (2D) Omega = (R^T dF - dF^T R)/tr S.

  z = KE(s_T) = 1/2 m_p sum_p |v_{T,p}|^2                     (final kinetic energy)
  lambda_T = dz/ds_T = (0, m_p v_T, 0, 0)
  lambda_t = G(s_t, lambda_{t+1}) = (ds_{t+1}/ds_t)^T lambda_{t+1}
  g_h = sum_{t=0..T} sum_p (lambda_{t,p,h})^2                 (Eq. 8)
Each state scalar (x_a, v_a, J, C_ab) is its own type h.

adjoint_step differentiates the forward exactly as written (piecewise: base = floor is
constant; a clamped out-of-domain fx (reading Q14) and a wall-clamped grid velocity
(reading Q13) have zero derivative; empty nodes carry none).

backward_bisection is the paper's bisection checkpointing (Griewank 1992):
to back-propagate over [lo, hi] from the state at lo, run forward to mid = (lo+hi)/2,
keep that checkpoint, back-propagate [mid, hi], drop it, then [lo, mid] -- O(log T)
resident states and O(T log T) forward steps.  backward_all stores every state.
"""
from __future__ import annotations

import numpy as np

import oracle


def _consts(sim):
    d = sim["dim"]
    dx = float(sim["dx"])
    E, nu = float(sim["E"]), float(sim["nu"])
    return dict(d=d, dx=dx, inv_dx=1.0 / dx, dt=float(sim["dt"]), m=float(sim["p_rho"] * sim["p_vol"]),
                k=-float(sim["dt"]) * float(sim["p_vol"]) * 4.0 / (dx * dx) * E,
                scale=-float(sim["dt"]) * float(sim["p_vol"]) * 4.0 / (dx * dx),
                mu=E / (2.0 * (1.0 + nu)), la=E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)),
                g=np.asarray(sim["gravity"][:d], dtype=np.float64), bound=int(sim["bound"]),
                res=np.asarray(sim["grid_res"][:d]))


def forward(sim, s):
    """One fp64 step s_t -> s_{t+1} (the C oracle)."""
    grid, origin, gsize, _ = oracle.p2g(sim, s)
    gv = oracle.grid_update(sim, grid, origin, gsize)
    return oracle.g2p(sim, s, gv, origin, gsize)


def kinetic_energy(sim, s):
    d = sim["dim"]
    m = float(sim["p_rho"] * sim["p_vol"])
    return 0.5 * m * float(np.sum(np.asarray(s, dtype=np.float64)[:, d:2 * d] ** 2))


def _base_fx(c, x):
    """base, fx and d fx / d x per axis with the out-of-domain clamp of reading Q14."""
    X = x * c["inv_dx"]
    base = np.floor(X - 0.5).astype(np.int64)
    oob = (base < 0) | (base > c["res"] - 3)
    base = np.clip(base, 0, c["res"] - 3)
    fx = X - base
    dfx = np.full(fx.shape, c["inv_dx"])
    lo, hi = oob & (fx < 0.5), oob & (fx > 1.5)
    fx = np.where(lo, 0.5, np.where(hi, 1.5, fx))
    dfx[lo | hi] = 0.0
    return base, fx, dfx


def _weights(fx):
    """Quadratic B-spline weights and their derivatives at offsets 0, 1, 2 (per axis)."""
    w = np.stack([0.5 * (1.5 - fx) ** 2, 0.75 - (fx - 1.0) ** 2, 0.5 * (fx - 0.5) ** 2], -1)
    dw = np.stack([-(1.5 - fx), -2.0 * (fx - 1.0), fx - 0.5], -1)
    return w, dw


def _offsets(d):
    if d == 2:
        return [(i, j) for i in range(3) for j in range(3)]
    return [(i, j, k) for i in range(3) for j in range(3) for k in range(3)]


def _polar(F):
    """R, S of F = R S (batched, det F > 0) by SVD."""
    U, sig, Vt = np.linalg.svd(F)
    R = U @ Vt
    S = np.einsum("pji,pj,pjk->pik", Vt, sig, Vt)
    return R, S


def _stress_F_adjoint(c, F, lP):
    """dL/dF for P F^T = 2 mu (F - R) F^T + lambda (J - 1) J I given dL/d(P F^T) = lP."""
    d = F.shape[1]
    mu, la = c["mu"], c["la"]
    R, S = _polar(F)
    J = np.linalg.det(F)
    lF = 2.0 * mu * (np.einsum("pab,pbc->pac", lP, F) + np.einsum("pba,pbc->pac", lP, F - R))
    lR = -2.0 * mu * np.einsum("pab,pbc->pac", lP, F)
    G = np.einsum("pba,pbc->pac", R, lR)  # R^T lR
    sk = 0.5 * (G - np.transpose(G, (0, 2, 1)))
    if d == 3:
        a = np.stack([sk[:, 2, 1], sk[:, 0, 2], sk[:, 1, 0]], -1)
        K = np.trace(S, axis1=1, axis2=2)[:, None, None] * np.eye(3)[None] - S
        cc = np.linalg.solve(K, a[..., None])[..., 0]
        X = np.zeros_like(F)
        X[:, 0, 1], X[:, 0, 2], X[:, 1, 2] = -cc[:, 2], cc[:, 1], -cc[:, 0]
        X[:, 1, 0], X[:, 2, 0], X[:, 2, 1] = cc[:, 2], -cc[:, 1], cc[:, 0]
        lF += 2.0 * np.einsum("pab,pbc->pac", R, X)
    else:
        lF += 2.0 * np.einsum("pab,pbc->pac", R, sk) / np.trace(S, axis1=1, axis2=2)[:, None, None]
    lJ = la * (2.0 * J - 1.0) * np.trace(lP, axis1=1, axis2=2)
    lF += (lJ * J)[:, None, None] * np.transpose(np.linalg.inv(F), (0, 2, 1))
    return lF


def _stress(c, F):
    R, _ = _polar(F)
    J = np.linalg.det(F)
    d = F.shape[1]
    PFt = 2.0 * c["mu"] * np.einsum("pab,pcb->pac", F - R, F) + (c["la"] * (J - 1.0) * J)[:, None, None] * np.eye(d)
    return c["scale"] * PFt


def adjoint_step(sim, s, lam_next):
    """lambda_t = (d s_{t+1} / d s_t)^T lambda_{t+1} (fp64), J-fluid or fixed-corotated."""
    fluid = sim["material"] == "fluid"
    c = _consts(sim)
    d, dx, inv_dx, dt, m, k = c["d"], c["dx"], c["inv_dx"], c["dt"], c["m"], c["k"]
    s = np.asarray(s, dtype=np.float64)
    lam1 = np.asarray(lam_next, dtype=np.float64)
    n = s.shape[0]
    nF = 1 if fluid else d * d
    x, v = s[:, :d], s[:, d:2 * d]
    C = s[:, 2 * d + nF:].reshape(n, d, d)
    lx1, lv1 = lam1[:, :d], lam1[:, d:2 * d]
    lC1 = lam1[:, 2 * d + nF:].reshape(n, d, d)
    if fluid:
        J, lJ1 = s[:, 2 * d], lam1[:, 2 * d]
    else:
        F, lF1 = s[:, 2 * d:2 * d + nF].reshape(n, d, d), lam1[:, 2 * d:2 * d + nF].reshape(n, d, d)

    # forward recompute: grid of step t
    grid, origin, gsize, _ = oracle.p2g(sim, s)
    gv = oracle.grid_update(sim, grid, origin, gsize)
    base, fx, dfx = _base_fx(c, x)
    w, dw = _weights(fx)
    offs = _offsets(d)

    def node(o):
        idx = [base[:, a] + o[a] - origin[a] for a in range(d)] + ([np.zeros(n, np.int64)] if d == 2 else [])
        return tuple(idx)

    def W_and_grad(o):
        W = np.ones(n)
        for a in range(d):
            W = W * w[:, a, o[a]]
        dW = np.zeros((n, d))
        for a in range(d):
            p = dw[:, a, o[a]].copy()
            for b in range(d):
                if b != a:
                    p = p * w[:, b, o[b]]
            dW[:, a] = p
        return W, dW

    # ---- G2P reverse: v' = sum W v_i, C' = 4 inv_dx sum W v_i (x) (o - fx),
    #      J' = J (1 + dt tr C'), x' = x + dt v'
    newC = np.zeros((n, d, d))
    for o in offs:
        W, _ = W_and_grad(o)
        vi = gv[node(o)][:, 1:1 + d]
        dpc = np.asarray(o, dtype=np.float64)[None, :] - fx
        newC += 4.0 * inv_dx * W[:, None, None] * vi[:, :, None] * dpc[:, None, :]
    lam = np.zeros_like(s)
    lx = lx1.copy()
    lv_tot = lv1 + dt * lx1
    if fluid:  # J' = J (1 + dt tr C')
        trC = np.trace(newC, axis1=1, axis2=2)
        lJ = lJ1 * (1.0 + dt * trC)
        lC_tot = lC1 + (lJ1 * J * dt)[:, None, None] * np.eye(d)[None]
    else:  # F' = (I + dt C') F
        Gm = np.eye(d)[None] + dt * newC
        lF = np.einsum("pba,pbc->pac", Gm, lF1)
        lC_tot = lC1 + dt * np.einsum("pab,pcb->pac", lF1, F)
    lfx = np.zeros((n, d))
    lgrid_v = np.zeros(gv.shape[:3] + (d,))
    for o in offs:
        W, dW = W_and_grad(o)
        ni = node(o)
        vi = gv[ni][:, 1:1 + d]
        dpc = np.asarray(o, dtype=np.float64)[None, :] - fx
        contrib = W[:, None] * (lv_tot + 4.0 * inv_dx * np.einsum("pab,pb->pa", lC_tot, dpc))
        np.add.at(lgrid_v, ni, contrib)
        lW = np.sum(lv_tot * vi, 1) + 4.0 * inv_dx * np.einsum("pab,pa,pb->p", lC_tot, vi, dpc)
        lfx += -4.0 * inv_dx * W[:, None] * np.einsum("pab,pa->pb", lC_tot, vi)
        lfx += lW[:, None] * dW

    # ---- grid reverse: v_i = P_i / m_i + dt g, wall-clamped (reading Q13)
    mass = grid[..., 0]
    P = grid[..., 1:1 + d]
    has = mass > 0
    safe_m = np.where(has, mass, 1.0)
    u = P / safe_m[..., None]
    vt = u + dt * c["g"]
    ijk = np.stack(np.meshgrid(*[origin[a] + np.arange(gsize[a]) for a in range(3)], indexing="ij"), -1)[..., :d]
    clamp = ((ijk < c["bound"]) & (vt < 0)) | ((ijk > c["res"] - c["bound"]) & (vt > 0))
    lvt = np.where(clamp | ~has[..., None], 0.0, lgrid_v)
    lP = lvt / safe_m[..., None]
    lm = -np.sum(lvt * u, -1) / safe_m

    # ---- P2G reverse: m_i += W m, P_i += W (m v + A dpos), A = stress + m C
    if fluid:
        A = (k * (J - 1.0))[:, None, None] * np.eye(d)[None] + m * C
    else:
        A = _stress(c, F) + m * C
    lv = np.zeros((n, d))
    lA = np.zeros((n, d, d))
    for o in offs:
        W, dW = W_and_grad(o)
        ni = node(o)
        lPi = lP[ni]
        lmi = lm[ni]
        dpos = (np.asarray(o, dtype=np.float64)[None, :] - fx) * dx
        q = m * v + np.einsum("pab,pb->pa", A, dpos)
        lW = lmi * m + np.sum(lPi * q, 1)
        lv += (W * m)[:, None] * lPi
        lA += W[:, None, None] * lPi[:, :, None] * dpos[:, None, :]
        ldpos = W[:, None] * np.einsum("pab,pa->pb", A, lPi)
        lfx += -dx * ldpos + lW[:, None] * dW
    lC = m * lA
    lx = lx + dfx * lfx
    lam[:, :d] = lx
    lam[:, d:2 * d] = lv
    if fluid:
        lam[:, 2 * d] = lJ + k * np.trace(lA, axis1=1, axis2=2)
    else:
        lam[:, 2 * d:2 * d + nF] = (lF + _stress_F_adjoint(c, F, c["scale"] * lA)).reshape(n, nF)
    lam[:, 2 * d + nF:] = lC.reshape(n, d * d)
    return lam


def lambda_T(sim, sT):
    d = sim["dim"]
    m = float(sim["p_rho"] * sim["p_vol"])
    lam = np.zeros_like(np.asarray(sT, dtype=np.float64))
    lam[:, d:2 * d] = m * np.asarray(sT, dtype=np.float64)[:, d:2 * d]
    return lam


def backward_all(sim, s0, T):
    """Store every state; returns (z, g[ns], lambda_0)."""
    states = [np.asarray(s0, dtype=np.float64)]
    for _ in range(T):
        states.append(forward(sim, states[-1]))
    lam = lambda_T(sim, states[T])
    g = np.sum(lam ** 2, 0)
    for t in range(T - 1, -1, -1):
        lam = adjoint_step(sim, states[t], lam)
        g += np.sum(lam ** 2, 0)
    return kinetic_energy(sim, states[T]), g, lam


def backward_bisection(sim, s0, T, stats=None):
    """The paper's bisection checkpointing; same results as backward_all.
    stats (dict, optional) receives max_resident (states held at once, s0 included) and
    forward_steps."""
    st = {"resident": 1, "max_resident": 1, "forward_steps": 0}
    g = None

    def fwd(s, k):
        for _ in range(k):
            s = forward(sim, s)
            st["forward_steps"] += 1
        return s

    def back(lo, hi, s_lo, lam_hi):
        nonlocal g
        if hi - lo == 1:
            lam = adjoint_step(sim, s_lo, lam_hi)
            g += np.sum(lam ** 2, 0)
            return lam
        mid = (lo + hi) // 2
        s_mid = fwd(s_lo, mid - lo)
        st["resident"] += 1
        st["max_resident"] = max(st["max_resident"], st["resident"])
        lam_mid = back(mid, hi, s_mid, lam_hi)
        st["resident"] -= 1
        return back(lo, mid, s_lo, lam_mid)

    s0 = np.asarray(s0, dtype=np.float64)
    sT = fwd(s0, T)
    z = kinetic_energy(sim, sT)
    lam = lambda_T(sim, sT)
    g = np.sum(lam ** 2, 0)
    if T > 0:
        st["resident"] += 1  # s_T is dropped once lambda_T is formed; count it while held
        st["max_resident"] = max(st["max_resident"], st["resident"])
        st["resident"] -= 1
        lam = back(0, T, s0, lam)
    if stats is not None:
        stats.update(max_resident=st["max_resident"], forward_steps=st["forward_steps"])
    return z, g, lam
