"""Seeded synthetic scenes shaped like the paper's workloads (input generation only).

This module holds NO arithmetic of the method (no codec, no MPM): it produces the
initial particle state (x, v, F = I or J = 1, C = 0) and the scene parameters.
Both the CUDA path (via the product API) and the CPU oracle (via the tests) are
fed from it; it imports neither.

Workloads:
  C1  2D elastic: 8 squares of 32x32 jittered lattice (6.25 ppc), 128^2, dt 2e-4
  C2  3D elastic: 8 cubes of 50^3 (8 ppc), 1,000,000 particles, 256^3, dt 2e-4 (T-large initial)
  C3  3D elastic: 32 cubes of 209^3 + one partial cube = 295,280,208 particles, 1024^3,
      dt 7.5e-5 (T-large final)
  C4  3D fluid dam-break: water block, 400M particles on 256^3 (~68 ppc), dt 1e-4
Jitter is +-0.25 of the lattice spacing from a counter-based integer hash of the
particle's global index, so any chunk of any scene can be generated independently,
identically with numpy (host) or torch (device).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK32 = 0xFFFFFFFF


# ---------------------------------------------------------------- hashing
def _wang32(x, xp):
    """Thomas Wang's 32-bit integer hash on int64 containers (values < 2^32)."""
    x = (x ^ 61) ^ (x >> 16)
    x = (x + (x << 3)) & MASK32
    x = x ^ (x >> 4)
    x = (x * 0x27D4EB2D) & MASK32
    x = x ^ (x >> 15)
    return x


def _uniform(idx, salt, xp):
    """U[0,1) in float64 from a 64-bit counter `idx` (int64 array) and a salt."""
    lo = idx & MASK32
    hi = (idx >> 32) & MASK32
    h = _wang32(_wang32(lo ^ (salt & MASK32), xp) ^ hi ^ ((salt >> 32) & MASK32), xp)
    return h.to(dtype=xp.float64) / 4294967296.0 if xp is not np else h.astype(np.float64) / 4294967296.0


# ---------------------------------------------------------------- scenes
@dataclass
class Box:
    origin: tuple
    counts: tuple
    spacing: float
    velocity: tuple
    n: int = -1  # particles taken in lattice order (-1 = all)
    # a smooth per-particle flow added to `velocity` (developed-state parity scenes):
    # swirl * sin(2 pi (x_{a+1} - o_{a+1}) / L_{a+1}) on axis a, minus conv * (x_a - centre_a)
    swirl: float = 0.0
    conv: float = 0.0

    def size(self):
        full = int(np.prod(self.counts))
        return full if self.n < 0 else min(self.n, full)


@dataclass
class Scene:
    name: str
    dim: int
    material: str
    sim: dict
    boxes: list = field(default_factory=list)
    seed: int = 0

    @property
    def n_particles(self):
        return sum(b.size() for b in self.boxes)

    @property
    def n_scalars(self):
        d = self.dim
        return 2 * d + (1 if self.material == "fluid" else d * d) + d * d

    def state_chunk(self, start, count, backend="numpy", device=None):
        """float32 [count][n_scalars] initial state of particles [start, start+count).
        Scalar order: x[d], v[d], F[d*d] (row-major, = I) or J (= 1), C[d*d] (= 0)."""
        if backend == "numpy":
            xp = np
        else:
            import torch as xp  # noqa: N813
        d = self.dim
        out_x, out_v = [], []
        first = 0
        for bi, b in enumerate(self.boxes):
            nb = b.size()
            lo, hi = max(start, first), min(start + count, first + nb)
            if lo < hi:
                if xp is np:
                    g = np.arange(lo, hi, dtype=np.int64)
                else:
                    g = xp.arange(lo, hi, dtype=xp.int64, device=device)
                l = g - first
                idx = []
                rem = l
                for a in reversed(range(d)):  # last axis fastest
                    idx.append(rem % b.counts[a])
                    rem = rem // b.counts[a]
                idx = idx[::-1]
                xs = []
                for a in range(d):
                    u = _uniform(g * 4 + a, self.seed * 0x100000001 + 0x51ED27, xp)
                    jit = (u - 0.5) * 0.5
                    if xp is np:
                        pos = b.origin[a] + (idx[a].astype(np.float64) + 0.5 + jit) * b.spacing
                    else:
                        pos = b.origin[a] + (idx[a].to(xp.float64) + 0.5 + jit) * b.spacing
                    xs.append(pos)
                out_x.append(xs)
                if b.swirl or b.conv:
                    L = [b.counts[a] * b.spacing for a in range(d)]
                    vel = []
                    for a in range(d):
                        nb_ = (a + 1) % d
                        ph = (xs[nb_] - b.origin[nb_]) * (2.0 * math.pi / L[nb_])
                        sw = np.sin(ph) if xp is np else xp.sin(ph)
                        vel.append(b.velocity[a] + b.swirl * sw - b.conv * (xs[a] - (b.origin[a] + 0.5 * L[a])))
                    out_v.append((hi - lo, vel))
                else:
                    out_v.append((hi - lo, b.velocity))
            first += nb
        ns = self.n_scalars
        if xp is np:
            st = np.zeros((count, ns), dtype=np.float32)
        else:
            st = xp.zeros((count, ns), dtype=xp.float32, device=device)
        row = 0
        for xs, (m, vel) in zip(out_x, out_v):
            for a in range(d):
                st[row:row + m, a] = xs[a].astype(np.float32) if xp is np else xs[a].to(xp.float32)
                if isinstance(vel[a], float):
                    st[row:row + m, d + a] = float(np.float32(vel[a]))
                else:
                    st[row:row + m, d + a] = vel[a].astype(np.float32) if xp is np else vel[a].to(xp.float32)
            row += m
        if self.material == "fluid":
            st[:, 2 * d] = 1.0
        else:
            for a in range(d):
                st[:, 2 * d + a * d + a] = 1.0
        return st

    def state(self, backend="numpy", device=None):
        return self.state_chunk(0, self.n_particles, backend, device)

    def zrange_runs(self, z_lo, z_hi, margin=0.3):
        """(start, count) runs of global particle indices whose LATTICE z position lies
        within [z_lo - margin*s, z_hi + margin*s) -- a superset of the particles whose
        jittered z lies in [z_lo, z_hi) (jitter is +-0.25 s).  3D boxes only."""
        runs = []
        first = 0
        for b in self.boxes:
            nb = b.size()
            nx, ny, nz = b.counts
            k0 = 0 if z_lo == -math.inf else max(0, int(math.floor((z_lo - b.origin[2]) / b.spacing - 0.5 - margin)))
            k1 = nz if z_hi == math.inf else min(nz, int(math.ceil((z_hi - b.origin[2]) / b.spacing - 0.5 + margin)) + 1)
            if k0 < k1:
                for ij in range(nx * ny):
                    lo = ij * nz + k0
                    if lo >= nb:
                        break
                    hi = min(ij * nz + k1, nb)
                    if runs and runs[-1][0] + runs[-1][1] == first + lo:
                        runs[-1] = (runs[-1][0], runs[-1][1] + hi - lo)
                    else:
                        runs.append((first + lo, hi - lo))
            first += nb
        return runs

    def state_zrange(self, z_lo, z_hi, backend="numpy", device=None, max_chunk=1 << 24):
        """Generator of (global_indices, state) chunks of the particles whose z lies in
        [z_lo, z_hi): exactly the rows of state() with that z, in index order."""
        runs = self.zrange_runs(z_lo, z_hi)
        pend = []
        tot = 0

        def flush(pend):
            if backend == "numpy":
                idx = np.concatenate([np.arange(a, a + c, dtype=np.int64) for a, c in pend])
                st = np.concatenate([self.state_chunk(a, c) for a, c in pend])
                z = st[:, 2]
                keep = (z >= np.float32(z_lo)) & (z < np.float32(z_hi))
                return idx[keep], st[keep]
            import torch
            idx = torch.cat([torch.arange(a, a + c, dtype=torch.int64, device=device) for a, c in pend])
            st = torch.cat([self.state_chunk(a, c, backend, device) for a, c in pend])
            z = st[:, 2]
            keep = (z >= float(np.float32(z_lo))) & (z < float(np.float32(z_hi)))
            return idx[keep], st[keep]

        for a, c in runs:
            while c > 0:
                take = min(c, max_chunk - tot)
                pend.append((a, take))
                tot += take
                a += take
                c -= take
                if tot >= max_chunk:
                    yield flush(pend)
                    pend, tot = [], 0
        if pend:
            yield flush(pend)


def _box_velocity(seed, box_index, dim, vmax):
    if vmax == 0:
        return tuple(0.0 for _ in range(dim))
    idx = np.array([box_index * 8 + a for a in range(dim)], dtype=np.int64)
    u = _uniform(idx, seed * 0x100000001 + 0xB0C5, np)
    return tuple(float((2.0 * ui - 1.0) * vmax) for ui in u)


def _sim(dim, material, res, dt, E, p_vol, bound=3, nu=0.2, rho=1.0, gravity=None):
    g = gravity if gravity is not None else ((0.0, -9.8) if dim == 2 else (0.0, -9.8, 0.0))
    return dict(dim=dim, material=material, grid_res=tuple(res) + (1,) * (3 - dim),
                dx=1.0 / res[0], dt=dt, gravity=tuple(g) + (0.0,) * (3 - dim),
                p_rho=rho, p_vol=p_vol, E=E, nu=nu, bound=bound)


def c1(seed=0):
    """2D elastic, 8 squares (side 0.1, 32x32 lattice = 6.25 ppc), two staggered rows."""
    spacing = 0.1 / 32
    boxes = []
    for row, (y0, xoff) in enumerate(((0.3, 0.1), (0.6, 0.2))):
        for c in range(4):
            boxes.append(Box((xoff + 0.2 * c, y0), (32, 32), spacing, (0.0, 0.0)))
    sim = _sim(2, "elastic", (128, 128), 2e-4, 100.0, spacing ** 2)
    return Scene("C1", 2, "elastic", sim, boxes, seed)


def c2(seed=0, cube=50, res=256):
    """3D elastic, 8 cubes (2x2x2) of cube^3 lattice at spacing dx/2 (8 ppc), v0 ~ U(-1,1)."""
    dx = 1.0 / res
    spacing = dx / 2
    boxes = []
    for i, x0 in enumerate((0.30, 0.55)):
        for j, y0 in enumerate((0.20, 0.45)):
            for k, z0 in enumerate((0.30, 0.55)):
                bi = i * 4 + j * 2 + k
                boxes.append(Box((x0, y0, z0), (cube,) * 3, spacing, _box_velocity(seed, bi, 3, 1.0)))
    sim = _sim(3, "elastic", (res,) * 3, 2e-4, 25.0, spacing ** 3)
    return Scene("C2", 3, "elastic", sim, boxes, seed)


C3_PARTICLES = 295_280_208


def c3(seed=0, n_target=C3_PARTICLES, cube=209):
    """3D elastic at 1024^3: 32 cubes (4x4x2) of 209^3 + a partial cube (T-large).
    n_target < full count truncates (cubes taken in order) for reduced-size runs."""
    res = 1024
    dx = 1.0 / res
    spacing = dx / 2
    boxes = []
    bi = 0
    for j, y0 in enumerate((0.10, 0.35)):
        for i, x0 in enumerate((0.06, 0.28, 0.50, 0.72)):
            for k, z0 in enumerate((0.06, 0.28, 0.50, 0.72)):
                boxes.append(Box((x0, y0, z0), (cube,) * 3, spacing, _box_velocity(seed, bi, 3, 0.5)))
                bi += 1
    boxes.append(Box((0.45, 0.62, 0.45), (cube,) * 3, spacing, _box_velocity(seed, bi, 3, 0.5)))
    left = n_target
    out = []
    for b in boxes:
        take = min(left, b.size())
        if take <= 0:
            break
        b.n = take
        out.append(b)
        left -= take
    sim = _sim(3, "elastic", (res,) * 3, 7.5e-5, 12.0, spacing ** 3)
    return Scene("C3", 3, "elastic", sim, out, seed)


def c4(seed=0, n_target=400_000_000, res=256, dt=1e-4, z_extent=1.0, E=100.0):
    """3D fluid dam-break: block x in [3dx, 0.5], y in [3dx, 0.7], z over [3dx, z_extent-3dx]
    (the full slab axis).  Lattice spacing chosen so the block holds >= n_target
    particles; exactly n_target are taken in lattice order.  At rest, J = 1, C = 0."""
    dx = 1.0 / res
    lo = 3 * dx
    L = (0.5 - lo, 0.7 - lo, z_extent - 2 * lo)
    vol = L[0] * L[1] * L[2]
    s = (vol / n_target) ** (1.0 / 3.0)
    while True:
        counts = tuple(max(1, int(math.floor(Li / s))) for Li in L)
        if counts[0] * counts[1] * counts[2] >= n_target:
            break
        s *= 0.999
    spacing = min(L[a] / counts[a] for a in range(3))
    box = Box((lo, lo, lo), counts, spacing, (0.0, 0.0, 0.0), n_target)
    res3 = (res, res, int(round(res * z_extent)))
    sim = _sim(3, "fluid", res3, dt, E, spacing ** 3)
    return Scene("C4", 3, "fluid", sim, [box], seed)


def dense_elastic(n_target, res=1024, seed=0):
    """Capacity probe scene: one elastic block at 8 ppc (spacing dx/2) filling x and z
    (3 cells from the walls) and as many y layers as n_target needs, at rest."""
    dx = 1.0 / res
    spacing = dx / 2
    lo = 3 * dx
    nxz = int((1.0 - 2 * lo) / spacing)
    ny = -(-n_target // (nxz * nxz))
    box = Box((lo, lo, lo), (nxz, ny, nxz), spacing, (0.0, 0.0, 0.0), n_target)
    sim = _sim(3, "elastic", (res,) * 3, 7.5e-5, 12.0, spacing ** 3)
    return Scene("DENSE", 3, "elastic", sim, [box], seed)


def small_elastic_3d(seed=0, cube=12, res=64, vmax=1.0):
    """Reduced C2-like scene for fast parity tests (several blocks, ragged tails)."""
    dx = 1.0 / res
    spacing = dx / 2
    boxes = [Box((0.30, 0.30, 0.30), (cube, cube, cube), spacing, _box_velocity(seed, 0, 3, vmax)),
             Box((0.52, 0.35, 0.41), (cube + 3, cube - 2, cube + 1), spacing,
                 _box_velocity(seed, 1, 3, vmax))]
    sim = _sim(3, "elastic", (res,) * 3, 2e-4, 25.0, spacing ** 3)
    return Scene("S3", 3, "elastic", sim, boxes, seed)


def small_fluid_3d(seed=0, res=64, n_target=60_000):
    sc = c4(seed, n_target=n_target, res=res, dt=2e-4, E=50.0)
    sc.name = "S4"
    return sc


def developed_fluid(seed=0, res=64, cells=(14, 12, 14), ppc_axis=4.1, swirl=1.5, conv=6.0, dt=2e-4, E=100.0):
    """High-density fluid block for developed-state parity (SURVEY §8(c) P2 at C4 density):
    `ppc_axis`^3 particles per cell (C4 has ~4.2^3 = 72 ppc), a smooth swirling and
    converging initial flow (|v| ~ 1-2 m/s) so that after ~100 steps the block holds
    compression (J != 1), pressure and shear (C != 0) -- the P2G's full per-cell segments
    (48 particles) then carry non-trivial momentum and stress."""
    dx = 1.0 / res
    spacing = dx / ppc_axis
    counts = tuple(int(round(c * ppc_axis)) for c in cells)
    origin = (0.25, 0.12, 0.25)
    box = Box(origin, counts, spacing, (0.3, -0.2, 0.1), -1, swirl, conv)
    sim = _sim(3, "fluid", (res,) * 3, dt, E, spacing ** 3)
    return Scene("DF", 3, "fluid", sim, [box], seed)


def colliding_elastic(seed=0, res=64, cube=14, v=1.5, dt=2e-4, E=25.0):
    """Two elastic cubes at 8 ppc (C3's density) driven into each other at +-v with a
    swirl, for developed-state parity: after ~100 steps they are in contact with F far
    from I."""
    dx = 1.0 / res
    spacing = dx / 2
    c = (cube,) * 3
    boxes = [Box((0.26, 0.30, 0.30), c, spacing, (v, 0.0, 0.2), -1, 0.5, 0.0),
             Box((0.26 + cube * spacing + 2.5 * dx, 0.31, 0.305), c, spacing, (-v, 0.1, -0.2), -1, 0.5, 0.0)]
    sim = _sim(3, "elastic", (res,) * 3, dt, E, spacing ** 3)
    return Scene("CE", 3, "elastic", sim, boxes, seed)


BY_NAME = {"c1": c1, "c2": c2, "c3": c3, "c4": c4}


# ---------------------------------------------------------------- smoke (f4)
SMOKE_VOXELS = 228_982_784  # the paper's large smoke run (T-large)


def smoke(res=(64, 64, 64), seed=0, dt=0.01, buoyancy=1.0, amp=0.5, modes=4, rho_blobs=4, p_amp=0.0,
          jacobi_iters=64):
    """A seeded smoke scene on a collocated grid (DESIGN.md §12 input recipe): dx = 1/ny
    (unit-height box), a smooth random velocity field (sum of `modes` random Fourier modes
    per component, max |u| <= amp), density blobs in [0, 1], pressure p_amp-scaled modes
    (0: the usual zero warm start), a source box at the bottom centre.  dt 0.01.
    Returns (params dict, u [nx,ny,nz,3] f32, p [nx,ny,nz] f32, rho [nx,ny,nz] f32)."""
    nx, ny, nz = res
    rng = np.random.default_rng(seed)
    x = [np.arange(n, dtype=np.float64) / n for n in res]
    X, Y, Z = np.meshgrid(*x, indexing="ij")

    def field(a):
        f = np.zeros(res)
        for _ in range(modes):
            k = rng.integers(1, 4, size=3)
            ph = rng.uniform(0, 2 * np.pi, size=3)
            f += rng.uniform(-1, 1) * np.sin(2 * np.pi * k[0] * X + ph[0]) * np.sin(2 * np.pi * k[1] * Y + ph[1]) \
                * np.sin(2 * np.pi * k[2] * Z + ph[2])
        m = np.abs(f).max()
        return (a * f / m if m > 0 else f).astype(np.float32)

    u = np.stack([field(amp) for _ in range(3)], -1) if amp > 0 else np.zeros(res + (3,), np.float32)
    p = field(p_amp) if p_amp > 0 else np.zeros(res, np.float32)
    rho = np.zeros(res)
    for _ in range(rho_blobs):
        c = rng.uniform(0.2, 0.8, size=3)
        r = rng.uniform(0.05, 0.2)
        rho += np.exp(-((X - c[0]) ** 2 + (Y - c[1]) ** 2 + (Z - c[2]) ** 2) / (r * r))
    rho = np.clip(rho, 0, 1).astype(np.float32)
    lo = (nx * 3 // 8, 1, nz * 3 // 8)
    hi = (max(lo[0] + 1, nx * 5 // 8), max(2, ny // 16 + 1), max(lo[2] + 1, nz * 5 // 8))
    params = dict(res=tuple(res), dx=1.0 / ny, dt=dt, buoyancy=buoyancy, source_lo=lo, source_hi=hi,
                  jacobi_iters=jacobi_iters)
    return params, u.astype(np.float32), p, rho


def smoke_plume(res, dt=0.01, buoyancy=1.0, jacobi_iters=64):
    """The large-scale bench scene: everything at rest, zero density, the source box at the
    bottom centre (the plume rises by buoyancy)."""
    params, u, p, rho = smoke(res=res, amp=0.0, rho_blobs=0, dt=dt, buoyancy=buoyancy, jacobi_iters=jacobi_iters)
    return params


# ---------------------------------------------------------------- adjoint (f3)
def adjoint_fluid(dim=2, side=8, res=32, seed=0, dt=2e-4, E=50.0, vmax=1.0, jitter=0.25, dJ=0.02, cmax=2.0,
                  ppc=2, origin=0.35, gravity=None):
    """A seeded J-fluid block for the gradient-tally path (DESIGN.md §13 input recipe):
    side^dim particles on a jittered lattice of spacing dx/ppc starting at `origin`
    (fraction of the box), random velocity |v_a| <= vmax, J = 1 + U(-dJ, dJ), C with
    entries U(-cmax, cmax).  Returns (sim, state [n][ns] float32)."""
    rng = np.random.default_rng(seed)
    sim = _sim(dim, "fluid", (res,) * dim, dt, E, p_vol=(1.0 / res / ppc) ** dim, gravity=gravity)
    h = sim["dx"] / ppc
    grid = np.stack(np.meshgrid(*[np.arange(side)] * dim, indexing="ij"), -1).reshape(-1, dim)
    x = origin + (grid + 0.5 + rng.uniform(-jitter, jitter, grid.shape)) * h
    n = x.shape[0]
    v = rng.uniform(-vmax, vmax, (n, dim))
    J = 1.0 + rng.uniform(-dJ, dJ, (n, 1))
    C = rng.uniform(-cmax, cmax, (n, dim * dim))
    return sim, np.concatenate([x, v, J, C], 1).astype(np.float32)


def adjoint_elastic(dim=2, side=8, res=32, seed=0, dt=2e-4, E=500.0, nu=0.2, vmax=1.0, jitter=0.25, dF=0.05,
                    cmax=2.0, ppc=2, origin=0.35, gravity=None):
    """A seeded fixed-corotated block for the gradient-tally path: as adjoint_fluid, with
    F = I + U(-dF, dF) per entry (det F > 0) instead of J.  Returns (sim, state float32)."""
    rng = np.random.default_rng(seed)
    sim = _sim(dim, "elastic", (res,) * dim, dt, E, p_vol=(1.0 / res / ppc) ** dim, nu=nu, gravity=gravity)
    h = sim["dx"] / ppc
    grid = np.stack(np.meshgrid(*[np.arange(side)] * dim, indexing="ij"), -1).reshape(-1, dim)
    x = origin + (grid + 0.5 + rng.uniform(-jitter, jitter, grid.shape)) * h
    n = x.shape[0]
    v = rng.uniform(-vmax, vmax, (n, dim))
    F = np.eye(dim).reshape(1, -1) + rng.uniform(-dF, dF, (n, dim * dim))
    C = rng.uniform(-cmax, cmax, (n, dim * dim))
    return sim, np.concatenate([x, v, F, C], 1).astype(np.float32)
