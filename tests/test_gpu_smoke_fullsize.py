"""Smoke parity at the bench's full size (612^3 = 229M voxels, bench_smoke.py's launch
configuration): every sub-step kernel runs once over the whole grid from seeded inputs,
and a sample of records (interior and on every wall) is checked against the oracle one
by one.  Inputs are separable analytic fields generated on the host and encoded by the
oracle codec; the oracle's input for a sampled record is the sub-box of those host
words around it (a margin of 4 cells: the departure points move less than one cell),
so nothing the oracle reads comes from the GPU."""
import numpy as np
import pytest

import oracle
from oracle import smoke as osm
from paper_2207_04658_b200 import qsmoke, scenes, schemes
from test_gpu_smoke import TOL

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")

RES = (612, 612, 612)
M = 4  # sub-box margin (cells)


def separable(res, seed, amp, modes=3):
    """f(x, y, z) = sum_m a_m sx_m(x) sy_m(y) sz_m(z) with sine factors: returns a
    chunk(x0, x1) -> float32 [x1 - x0, ny, nz] generator (identical for any chunking)."""
    rng = np.random.default_rng(seed)
    facs = []
    for _ in range(modes):
        a = rng.uniform(-1, 1)
        f = [np.sin(2 * np.pi * rng.integers(1, 4) * np.arange(n) / n + rng.uniform(0, 2 * np.pi)) for n in res]
        facs.append((a, f))
    norm = amp / sum(abs(a) for a, _ in facs)

    def chunk(x0, x1):
        out = np.zeros((x1 - x0,) + tuple(res[1:]))
        for a, (fx, fy, fz) in facs:
            out += a * fx[x0:x1, None, None] * (fy[:, None] * fz[None, :])[None]
        return (out * norm).astype(np.float32)
    return chunk


def encode_field(chunks, scheme, res, dstep, xs=36):
    """Encode comps = len(chunks) fields into records (oracle codec), x-slab by x-slab."""
    nx, ny, nz = res
    comps = len(chunks)
    out = []
    for x0 in range(0, nx, xs):
        x1 = min(nx, x0 + xs)
        f = np.stack([c(x0, x1) for c in chunks], -1)
        rec = osm.to_records(f, comps)
        r0 = (x0 // 2) * ny * nz
        keys = np.arange(r0, r0 + rec.shape[0], dtype=np.uint32)
        w, _ = oracle.encode(scheme, rec, keys=keys, step=dstep)
        out.append(w)
    return np.concatenate(out)


def box(words, scheme, comps, res, xr, y, z, m=M):
    """Decoded sub-box of a record field around record (xr, y, z): cells x in
    [2xr - m, 2xr + 2 + m) (even-aligned), y, z within +-m, clipped to the domain.
    Returns (field [bx, by, bz, comps], (x0, y0, z0))."""
    nx, ny, nz = res
    x0, x1 = max(0, 2 * xr - m), min(nx, 2 * xr + 2 + m)
    y0, y1 = max(0, y - m), min(ny, y + m + 1)
    z0, z1 = max(0, z - m), min(nz, z + m + 1)
    xr0, xr1 = x0 // 2, x1 // 2
    W = words.shape[1]
    w3 = words.reshape(nx // 2, ny, nz, W)[xr0:xr1, y0:y1, z0:z1]
    dec = oracle.decode(scheme, w3.reshape(-1, W)).astype(np.float64)
    sub = dec.reshape(xr1 - xr0, y1 - y0, z1 - z0, 2, comps).transpose(0, 3, 1, 2, 4)
    return sub.reshape(2 * (xr1 - xr0), y1 - y0, z1 - z0, comps), (2 * xr0, y0, z0)


def sample_records(res, n=40, seed=11):
    nx, ny, nz = res
    rng = np.random.default_rng(seed)
    pts = [(rng.integers(0, nx // 2), rng.integers(0, ny), rng.integers(0, nz)) for _ in range(n)]
    pts += [(0, 0, 0), (nx // 2 - 1, ny - 1, nz - 1), (0, ny // 2, nz - 1), (nx // 2 - 1, 0, nz // 3),
            (nx // 4, ny - 1, 0), (nx // 3, 5, nz - 1)]
    return [tuple(int(v) for v in p) for p in pts]


@pytest.fixture(scope="module")
def state():
    res = RES
    su, sp = schemes.smoke_u(), schemes.smoke_p()
    params = scenes.smoke_plume(res)
    u_gen = [separable(res, 100 + c, 0.4) for c in range(3)]
    ur_gen = [separable(res, 200 + c, 0.4) for c in range(3)]
    p_gen = separable(res, 300, 0.02)
    d_gen = separable(res, 400, 5.0)
    rho_gen = separable(res, 500, 1.0)
    uw = encode_field(u_gen, su, res, 255)
    urw = encode_field(ur_gen, su, res, 254)
    pw = encode_field([p_gen], sp, res, 253)
    div = np.concatenate([d_gen(x0, min(res[0], x0 + 64)) for x0 in range(0, res[0], 64)])
    rho = np.abs(np.concatenate([rho_gen(x0, min(res[0], x0 + 64)) for x0 in range(0, res[0], 64)]))
    return dict(res=res, su=su, sp=sp, params=params, uw=uw, urw=urw, pw=pw, div=div, rho=rho)


def dev(a):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).cuda()


def rec_index(res, xr, y, z):
    return (xr * res[1] + y) * res[2] + z


def test_fullsize_advection_sampled(state):
    res, su, sp, params = state["res"], state["su"], state["sp"], state["params"]
    dx, dt = params["dx"], params["dt"]
    bdt = 0.5 * dt * params["buoyancy"]
    sm = qsmoke.Smoke(params, su, sp)
    n = sm.n_records
    U, UR, RHO = dev(state["uw"]), dev(state["urw"]), dev(state["rho"])
    out = torch.empty((n, sm.Wu), dtype=torch.int32, device="cuda")
    dbg = torch.empty((n, 6), dtype=torch.float32, device="cuda")
    pts = sample_records(res)
    idx = torch.tensor([rec_index(res, *p) for p in pts], device="cuda")
    for refl in (False, True):
        ds = 9 * 256 + (100 if refl else 0)
        if refl:
            sm.advect_velocity(U, out, 0.5 * dt, u_refl=UR, dstep=ds, dbg=dbg)
        else:
            sm.advect_velocity(U, out, 0.5 * dt, rho=RHO, bdt=bdt, dstep=ds, dbg=dbg)
        g_pre = dbg[idx].cpu().numpy()
        g_w = out[idx].cpu().numpy().view(np.uint32)
        for q, (xr, y, z) in enumerate(pts):
            ub, (x0, y0, z0) = box(state["uw"], su, 3, res, xr, y, z)
            pos = osm.backtrace(ub, 0.5 * dt, dx)
            if refl:
                qb, _ = box(state["urw"], su, 3, res, xr, y, z)
                field = 2.0 * ub - qb
            else:
                field = ub
            o = np.zeros(6)
            for c in range(2):
                cx, cy, cz = 2 * xr + c - x0, y - y0, z - z0
                v = osm.sample(field, pos[cx, cy, cz][None])[0]
                if not refl:
                    v[1] += bdt * float(state["rho"][2 * xr + c, y, z])
                o[3 * c:3 * c + 3] = v
            scale = max(np.abs(ub).max(), 1e-6)
            assert np.abs(g_pre[q] - o).max() <= TOL * scale, (refl, (xr, y, z), g_pre[q], o)
        keys_ok = np.array([rec_index(res, *p) for p in pts], dtype=np.uint32)
        w_ref, _ = oracle.encode(su, g_pre, keys=keys_ok, step=ds)
        assert np.array_equal(g_w, w_ref), refl
    sm.close()


def test_fullsize_stencils_sampled(state):
    res, su, sp, params = state["res"], state["su"], state["sp"], state["params"]
    dx = params["dx"]
    sm = qsmoke.Smoke(params, su, sp)
    n = sm.n_records
    U, P, DIV = dev(state["uw"]), dev(state["pw"]), dev(state["div"])
    pts = sample_records(res, seed=12)
    idx = torch.tensor([rec_index(res, *p) for p in pts], device="cuda")
    keys = np.array([rec_index(res, *p) for p in pts], dtype=np.uint32)
    # divergence (fp32 per cell)
    dv = torch.empty(res, dtype=torch.float32, device="cuda")
    sm.divergence(U, dv)
    g_div = dv.cpu().numpy()
    # Jacobi sweep from the host div field
    pout = torch.empty((n, sm.Wp), dtype=torch.int32, device="cuda")
    dbg_p = torch.empty((n, 2), dtype=torch.float32, device="cuda")
    sm.jacobi(P, DIV, pout, dstep=9 * 256 + 7, dbg=dbg_p)
    gp_pre, gp_w = dbg_p[idx].cpu().numpy(), pout[idx].cpu().numpy().view(np.uint32)
    # projection
    uout = torch.empty((n, sm.Wu), dtype=torch.int32, device="cuda")
    dbg_u = torch.empty((n, 6), dtype=torch.float32, device="cuda")
    sm.project(U, P, uout, dstep=9 * 256 + 1, dbg=dbg_u)
    gu_pre, gu_w = dbg_u[idx].cpu().numpy(), uout[idx].cpu().numpy().view(np.uint32)
    for q, (xr, y, z) in enumerate(pts):
        ub, (x0, y0, z0) = box(state["uw"], su, 3, res, xr, y, z, m=2)
        pb, _ = box(state["pw"], sp, 1, res, xr, y, z, m=2)
        pb = pb[..., 0]
        # sub-box faces inside the domain are not walls, so S5-S7 are wrong on them; the
        # centre cells (m = 2 cells in) see only true data
        dvb = osm.divergence(ub, dx)
        dsub = state["div"][x0:x0 + ub.shape[0], y0:y0 + ub.shape[1], z0:z0 + ub.shape[2]].astype(np.float64)
        jb = osm.jacobi_sweep(pb, dsub, dx)
        gr = osm.gradient(pb, dx)
        for c in range(2):
            cx, cy, cz = 2 * xr + c - x0, y - y0, z - z0
            o_div = dvb[cx, cy, cz]
            assert abs(g_div[2 * xr + c, y, z] - o_div) <= TOL * max(np.abs(dvb).max(), 1e-6), ("div", (xr, y, z))
            assert abs(gp_pre[q, c] - jb[cx, cy, cz]) <= TOL * max(np.abs(jb).max(), 1e-6), ("jacobi", (xr, y, z))
            v = ub[cx, cy, cz] - gr[cx, cy, cz]
            X, Y, Z = 2 * xr + c, y, z
            if X == 0 or X == res[0] - 1:
                v[0] = 0.0
            if Y == 0 or Y == res[1] - 1:
                v[1] = 0.0
            if Z == 0 or Z == res[2] - 1:
                v[2] = 0.0
            assert np.abs(gu_pre[q, 3 * c:3 * c + 3] - v).max() <= TOL * max(np.abs(ub).max(), 1e-6), \
                ("project", (xr, y, z))
    w_ref, _ = oracle.encode(sp, gp_pre, keys=keys, step=9 * 256 + 7)
    assert np.array_equal(gp_w, w_ref)
    w_ref, _ = oracle.encode(su, gu_pre, keys=keys, step=9 * 256 + 1)
    assert np.array_equal(gu_w, w_ref)
    sm.close()


def test_fullsize_density_sampled(state):
    res, su, sp, params = state["res"], state["su"], state["sp"], state["params"]
    dx, dt = params["dx"], params["dt"]
    sm = qsmoke.Smoke(params, su, sp)
    U, RHO = dev(state["uw"]), dev(state["rho"])
    out = torch.empty(res, dtype=torch.float32, device="cuda")
    sm.advect_density(RHO, U, out, dt)
    g = out.cpu().numpy()
    lo, hi = params["source_lo"], params["source_hi"]
    for (xr, y, z) in sample_records(res, seed=13) + [(lo[0] // 2, lo[1], lo[2])]:
        ub, (x0, y0, z0) = box(state["uw"], su, 3, res, xr, y, z)
        rb = state["rho"][x0:x0 + ub.shape[0], y0:y0 + ub.shape[1], z0:z0 + ub.shape[2]].astype(np.float64)
        pos = osm.backtrace(ub, dt, dx)
        for c in range(2):
            X = 2 * xr + c
            if lo[0] <= X < hi[0] and lo[1] <= y < hi[1] and lo[2] <= z < hi[2]:
                o = 1.0
            else:
                o = osm.sample(rb, pos[X - x0, y - y0, z - z0][None])[0]
            assert abs(g[X, y, z] - o) <= TOL * max(np.abs(rb).max(), 1e-6), ((xr, y, z), c, g[X, y, z], o)
    sm.close()
