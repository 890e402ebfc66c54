"""Oracle of the quantized Eulerian smoke step -- numpy, fp64.

TEST INFRASTRUCTURE ONLY (same rule as the rest of oracle/).  It shares no code with
paper_2207_04658_b200/csrc/smoke*.  The codec steps call the C oracle codec
(oracle.encode / oracle.decode).

The paper's smoke solver: advection-reflection
(Zehnder et al. 2018, cited P:561), semi-Lagrangian advection with RK-3 path
integration, Poisson's equation by 64 Jacobi iterations, quantized pressure and
velocity on the grid.  The paper gives nothing more; the readings (DESIGN.md §12,
"S1".."S8") are restated where used:
  S1 grid: collocated (cell-centred) nx x ny x nz cells of size dx = 1/nx; u in world
     units per second; positions in cell units (cell c's centre at c).
  S2 records: two cells along x per record (x = 2r, 2r+1), fields in order
     cell0 comps, cell1 comps; u records 6 fields, p records 2 fields (bit pack).
  S3 sampling: trilinear, positions clamped to [0, n-1] per axis (clamp to edge).
  S4 RK-3 backtrace (Ralston): k1 = u(x), k2 = u(x - dt/2 k1), k3 = u(x - 3dt/4 k2),
     x_back = x - dt (2/9 k1 + 1/3 k2 + 4/9 k3)  (k in cells per second: u / dx).
  S5 divergence: central differences (u_{i+1} - u_{i-1}) / (2 dx), u = 0 outside.
  S6 Jacobi: p_i <- (sum of the 6 neighbours' p - dx^2 div_i) / 6, a neighbour outside
     the domain contributes p_i (Neumann); 64 sweeps from the stored p (warm start).
  S7 projection: u -= grad p, central differences (p_{i+1} - p_{i-1}) / (2 dx) with the
     same Neumann rule; then the wall-normal component of u is zeroed in the boundary
     layer of cells.
  S8 step (advection-reflection): u~ = A(u, u, dt/2) + dt/2 b rho e_y;  u_h = P(u~);
     u^ = 2 u_h - u~;  u' = A(u^, u_h, dt/2);  u_new = P(u');  rho_new = A(rho, u_new, dt),
     then rho = 1 in the source box.  Every store of u or p is encoded (dithered with
     the record index as key, salt of (step, sub-step), reading Q5); rho is fp32 (P:579:
     "the quantized variables are the pressure and velocity").
"""
from __future__ import annotations

import numpy as np

import oracle

JACOBI_ITERS = 64


def salt_step(step, sub):
    """Dither stream of sub-step `sub` of step `step` (S8): step index = step * 256 + sub."""
    return step * 256 + sub


def to_records(field, comps):
    """[nx, ny, nz, comps] -> [n_records, 2 * comps] (S2: cells x = 2r, 2r+1 of a record)."""
    nx, ny, nz = field.shape[:3]
    f = field.reshape(nx // 2, 2, ny, nz, comps).transpose(0, 2, 3, 1, 4)
    return np.ascontiguousarray(f.reshape(-1, 2 * comps))


def from_records(rec, shape, comps):
    nx, ny, nz = shape
    f = rec.reshape(nx // 2, ny, nz, 2, comps).transpose(0, 3, 1, 2, 4)
    return np.ascontiguousarray(f.reshape(nx, ny, nz, comps))


def store(field, scheme, step, sub, comps):
    """Encode a field (dithered, keys = record index) and return (words, decoded field)."""
    shape = field.shape[:3]
    vals = to_records(field.reshape(shape + (comps,)), comps).astype(np.float32)
    keys = np.arange(vals.shape[0], dtype=np.uint32)
    words, _ = oracle.encode(scheme, vals, keys=keys, step=salt_step(step, sub))
    return words, decode(words, scheme, shape, comps)


def decode(words, scheme, shape, comps):
    return from_records(oracle.decode(scheme, words).astype(np.float64), shape, comps)


def sample(f, pos):
    """Trilinear sample of cell-centred field f [nx, ny, nz, ...] at positions pos
    [..., 3] in cell units, clamped to the domain (S3)."""
    n = np.array(f.shape[:3])
    p = np.clip(pos, 0.0, n - 1.0)
    i0 = np.minimum(np.floor(p).astype(np.int64), n - 2)
    t = p - i0
    out = 0.0
    for dx_ in (0, 1):
        for dy_ in (0, 1):
            for dz_ in (0, 1):
                w = ((t[..., 0] if dx_ else 1 - t[..., 0]) * (t[..., 1] if dy_ else 1 - t[..., 1]) *
                     (t[..., 2] if dz_ else 1 - t[..., 2]))
                v = f[i0[..., 0] + dx_, i0[..., 1] + dy_, i0[..., 2] + dz_]
                out = out + (w[..., None] * v if v.ndim > w.ndim else w * v)
    return out


def backtrace(u, dt, dx):
    """RK-3 (Ralston) departure points of every cell centre (S4)."""
    nx, ny, nz = u.shape[:3]
    x = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1).astype(np.float64)
    k1 = sample(u, x) / dx
    k2 = sample(u, x - 0.5 * dt * k1) / dx
    k3 = sample(u, x - 0.75 * dt * k2) / dx
    return x - dt * (2.0 / 9.0 * k1 + 1.0 / 3.0 * k2 + 4.0 / 9.0 * k3)


def advect(q, u, dt, dx):
    """Semi-Lagrangian advection of q by u over dt (S4, S3)."""
    return sample(q, backtrace(u, dt, dx))


def _shift(f, axis, d, fill):
    """f shifted so out[i] = f[i + d] along axis; outside the domain -> fill (array or 0)."""
    out = np.roll(f, -d, axis=axis)
    idx = [slice(None)] * f.ndim
    idx[axis] = slice(-1, None) if d > 0 else slice(0, 1)
    out[tuple(idx)] = fill[tuple(idx)] if isinstance(fill, np.ndarray) else fill
    return out


def divergence(u, dx):
    """Central differences, u = 0 outside the domain (S5)."""
    div = 0.0
    for a in range(3):
        div = div + (_shift(u[..., a], a, 1, 0.0) - _shift(u[..., a], a, -1, 0.0)) / (2 * dx)
    return div


def jacobi_sweep(p, div, dx):
    """One Jacobi sweep with Neumann walls (S6)."""
    s = 0.0
    for a in range(3):
        s = s + _shift(p, a, 1, p) + _shift(p, a, -1, p)
    return (s - dx * dx * div) / 6.0


def gradient(p, dx):
    """Central differences with the Neumann rule (S7)."""
    return np.stack([(_shift(p, a, 1, p) - _shift(p, a, -1, p)) / (2 * dx) for a in range(3)], -1)


def zero_walls(u):
    """Wall-normal velocity zeroed in the boundary layer of cells (S7)."""
    u = u.copy()
    u[0, :, :, 0] = 0.0
    u[-1, :, :, 0] = 0.0
    u[:, 0, :, 1] = 0.0
    u[:, -1, :, 1] = 0.0
    u[:, :, 0, 2] = 0.0
    u[:, :, -1, 2] = 0.0
    return u


def project(u, p_words, scheme_u, scheme_p, step, sub0, dx, iters=JACOBI_ITERS, record=None):
    """S6-S7 with every store quantized: div (fp32 in the GPU path, fp64 here), `iters`
    Jacobi sweeps each storing p (sub-steps sub0 + 1 ..), then u -= grad p, walls, and
    the store of u (sub-step sub0).  Returns (u_words, u, p_words, p)."""
    shape = u.shape[:3]
    div = divergence(u, dx)
    p = decode(p_words, scheme_p, shape, 1)[..., 0]
    for k in range(iters):
        pn = jacobi_sweep(p, div, dx)
        if record is not None:
            record.append(("p", sub0 + 1 + k, pn))
        p_words, pq = store(pn[..., None], scheme_p, step, sub0 + 1 + k, 1)
        p = pq[..., 0]
    un = zero_walls(u - gradient(p, dx))
    if record is not None:
        record.append(("u", sub0, un))
    u_words, uq = store(un, scheme_u, step, sub0, 3)
    return u_words, uq, p_words, p


def step(state, params, scheme_u, scheme_p, step_index, iters=JACOBI_ITERS, record=None):
    """One advection-reflection step (S8).  state = (u_words, p_words, rho fp32 array).
    Sub-steps: 0 first advection, 1 first projection (+ 2..iters+1 its sweeps),
    100 second advection, 101 second projection (+ 102..)."""
    u_words, p_words, rho = state
    shape = tuple(params["res"])
    dx, dt, b = params["dx"], params["dt"], params["buoyancy"]
    u = decode(u_words, scheme_u, shape, 3)
    # 1. u~ = A(u, u, dt/2) + dt/2 b rho e_y
    ut = advect(u, u, 0.5 * dt, dx)
    ut[..., 1] += 0.5 * dt * b * rho.astype(np.float64)
    if record is not None:
        record.append(("u", 0, ut))
    ut_words, utq = store(ut, scheme_u, step_index, 0, 3)
    # 2. u_h = P(u~)
    uh_words, uh, p_words, _ = project(utq, p_words, scheme_u, scheme_p, step_index, 1, dx, iters, record)
    # 3.-4. u' = A(2 u_h - u~, u_h, dt/2)
    uhat = 2.0 * uh - utq
    up = sample(uhat, backtrace(uh, 0.5 * dt, dx))
    if record is not None:
        record.append(("u", 100, up))
    up_words, upq = store(up, scheme_u, step_index, 100, 3)
    # 5. u_new = P(u')
    un_words, un, p_words, _ = project(upq, p_words, scheme_u, scheme_p, step_index, 101, dx, iters, record)
    # 6. rho (fp32) advected by u_new over dt, then the source box
    rho_n = advect(rho.astype(np.float64), un, dt, dx).astype(np.float32)
    lo, hi = params["source_lo"], params["source_hi"]
    rho_n[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = 1.0
    return un_words, p_words, rho_n
