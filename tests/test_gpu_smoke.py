"""GPU parity of the quantized smoke step (include/qsmoke.h) against the
oracle (oracle/smoke.py), through the C-ABI.

Each sub-step kernel runs from oracle-encoded inputs and is checked twice: its values
before encoding (dbg) against the oracle's fp64 values within TOL of the field's scale
(fp32 arithmetic: DESIGN.md §12), and its output words bit-exactly against the oracle's
encoding of those same values (the dither decision is the codec's, keyed by record and
dither step).  The whole step (the CUDA graph of qsmoke_step) is then checked bit-exactly
against the chain of sub-step calls, each link of which is checked against the oracle
on the GPU's own inputs."""
import numpy as np
import pytest

import oracle
from oracle import smoke as osm
from paper_2207_04658_b200 import qsmoke, scenes, schemes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL = 2e-5  # |gpu - oracle| <= TOL * max |oracle| (fp32 vs fp64 on identical inputs)


def dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def host_u32(t):
    return t.cpu().numpy().view(np.uint32)


def check_close(g, o, what):
    scale = max(float(np.abs(o).max()), 1e-6)
    err = float(np.abs(g.astype(np.float64) - o).max())
    assert err <= TOL * scale, (what, err, scale)


def check_words(g_words, g_pre, scheme, dstep, what):
    keys = np.arange(g_pre.shape[0], dtype=np.uint32)
    w_ref, _ = oracle.encode(scheme, g_pre.astype(np.float32), keys=keys, step=dstep)
    bad = np.nonzero((g_words != w_ref).any(1))[0]
    assert bad.size == 0, (what, bad[:8], g_words[bad[:2]], w_ref[bad[:2]])


def make(res, seed=0, su=None, sp=None, iters=4, p_amp=0.05, **kw):
    params, u, p, rho = scenes.smoke(res=res, seed=seed, jacobi_iters=iters, p_amp=p_amp, **kw)
    su = su or schemes.smoke_u()
    sp = sp or schemes.smoke_p()
    uw, uq = osm.store(u.astype(np.float64), su, 0, 255, 3)
    pw, pq = osm.store(p[..., None].astype(np.float64), sp, 0, 255, 1)
    return params, su, sp, uw, uq, pw, pq[..., 0], rho


RES = [(16, 12, 10), (18, 7, 11), (2, 2, 2), (20, 10, 40)]  # several y and z tiles, ragged x marches


@pytest.mark.parametrize("res", RES)
def test_advect_velocity_parity(res):
    params, su, sp, uw, uq, pw, pq, rho = make(res, seed=1)
    sm = qsmoke.Smoke(params, su, sp)
    n, dx, dt = sm.n_records, params["dx"], params["dt"]
    bdt = 0.5 * dt * params["buoyancy"]
    for refl in (False, True):
        out = torch.zeros((n, sm.Wu), dtype=torch.int32, device="cuda")
        dbg = torch.zeros((n, 6), dtype=torch.float32, device="cuda")
        if refl:  # u' = A(2 u_h - u~, u_h): u_h = uq, u~ = a second field
            _, _, _, uw2, uq2, _, _, _ = make(res, seed=2)
            sm.advect_velocity(dev(uw), out, 0.5 * dt, u_refl=dev(uw2), dstep=7 * 256 + 100, dbg=dbg)
            o = osm.sample(2.0 * uq - uq2, osm.backtrace(uq, 0.5 * dt, dx))
            ds = 7 * 256 + 100
        else:
            sm.advect_velocity(dev(uw), out, 0.5 * dt, rho=dev(rho), bdt=bdt, dstep=7 * 256, dbg=dbg)
            o = osm.advect(uq, uq, 0.5 * dt, dx)
            o[..., 1] += bdt * rho.astype(np.float64)
            ds = 7 * 256
        g_pre = dbg.cpu().numpy()
        check_close(g_pre, osm.to_records(o, 3), ("advect", refl))
        check_words(host_u32(out), g_pre, su, ds, ("advect", refl))
    sm.close()


@pytest.mark.parametrize("res", RES)
def test_divergence_jacobi_project_parity(res):
    params, su, sp, uw, uq, pw, pq, rho = make(res, seed=3)
    sm = qsmoke.Smoke(params, su, sp)
    n, dx = sm.n_records, params["dx"]
    div = torch.zeros(res, dtype=torch.float32, device="cuda")
    sm.divergence(dev(uw), div)
    o_div = osm.divergence(uq, dx)
    check_close(div.cpu().numpy(), o_div, "div")
    # Jacobi from the oracle's fp32 divergence (both sides read the same fp32 array)
    d32 = o_div.astype(np.float32)
    pout = torch.zeros((n, sm.Wp), dtype=torch.int32, device="cuda")
    dbg = torch.zeros((n, 2), dtype=torch.float32, device="cuda")
    sm.jacobi(dev(pw), dev(d32), pout, dstep=3 * 256 + 5, dbg=dbg)
    o = osm.jacobi_sweep(pq, d32.astype(np.float64), dx)
    g_pre = dbg.cpu().numpy()
    check_close(g_pre, osm.to_records(o[..., None], 1), "jacobi")
    check_words(host_u32(pout), g_pre, sp, 3 * 256 + 5, "jacobi")
    # projection
    uout = torch.zeros((n, sm.Wu), dtype=torch.int32, device="cuda")
    dbg = torch.zeros((n, 6), dtype=torch.float32, device="cuda")
    sm.project(dev(uw), dev(pw), uout, dstep=3 * 256 + 1, dbg=dbg)
    o = osm.zero_walls(uq - osm.gradient(pq, dx))
    g_pre = dbg.cpu().numpy()
    check_close(g_pre, osm.to_records(o, 3), "project")
    check_words(host_u32(uout), g_pre, su, 3 * 256 + 1, "project")
    sm.close()


@pytest.mark.parametrize("res", RES)
def test_advect_density_parity(res):
    params, su, sp, uw, uq, pw, pq, rho = make(res, seed=4)
    sm = qsmoke.Smoke(params, su, sp)
    out = torch.zeros(res, dtype=torch.float32, device="cuda")
    sm.advect_density(dev(rho), dev(uw), out, params["dt"])
    o = osm.advect(rho.astype(np.float64), uq, params["dt"], params["dx"])
    lo, hi = params["source_lo"], params["source_hi"]
    o[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = 1.0
    check_close(out.cpu().numpy(), o, "rho")
    sm.close()


def chained_step(sm, params, su, sp, uw, pw, rho, step, iters):
    """One step as the chain of sub-step calls, each link checked against the oracle on
    the GPU's own inputs; returns the new (u words, p words, rho) as device tensors."""
    n, dx, dt = sm.n_records, params["dx"], params["dt"]
    res = params["res"]
    bdt = 0.5 * dt * params["buoyancy"]
    dbg_u = torch.zeros((n, 6), dtype=torch.float32, device="cuda")
    dbg_p = torch.zeros((n, 2), dtype=torch.float32, device="cuda")

    def dec_u(t):
        return osm.decode(host_u32(t), su, res, 3)

    def dec_p(t):
        return osm.decode(host_u32(t), sp, res, 1)[..., 0]

    def advect(uvel, urefl, rho_in, sub, out):
        sm.advect_velocity(uvel, out, 0.5 * dt, u_refl=urefl, rho=rho_in, bdt=bdt if rho_in is not None else 0.0,
                           dstep=step * 256 + sub, dbg=dbg_u)
        uv = dec_u(uvel)
        q = uv if urefl is None else 2.0 * uv - dec_u(urefl)
        o = osm.sample(q, osm.backtrace(uv, 0.5 * dt, dx))
        if rho_in is not None:
            o[..., 1] += bdt * rho_in.cpu().numpy().astype(np.float64)
        g = dbg_u.cpu().numpy()
        check_close(g, osm.to_records(o, 3), ("advect", step, sub))
        check_words(host_u32(out), g, su, step * 256 + sub, ("advect", step, sub))

    def projection(u_in, p, sub0, out):
        div = torch.zeros(res, dtype=torch.float32, device="cuda")
        sm.divergence(u_in, div)
        check_close(div.cpu().numpy(), osm.divergence(dec_u(u_in), dx), ("div", step, sub0))
        for k in range(iters):
            pn = torch.zeros_like(p)
            sm.jacobi(p, div, pn, dstep=step * 256 + sub0 + 1 + k, dbg=dbg_p)
            o = osm.jacobi_sweep(dec_p(p), div.cpu().numpy().astype(np.float64), dx)
            g = dbg_p.cpu().numpy()
            check_close(g, osm.to_records(o[..., None], 1), ("jacobi", step, sub0, k))
            check_words(host_u32(pn), g, sp, step * 256 + sub0 + 1 + k, ("jacobi", step, sub0, k))
            p = pn
        sm.project(u_in, p, out, dstep=step * 256 + sub0, dbg=dbg_u)
        o = osm.zero_walls(dec_u(u_in) - osm.gradient(dec_p(p), dx))
        g = dbg_u.cpu().numpy()
        check_close(g, osm.to_records(o, 3), ("project", step, sub0))
        check_words(host_u32(out), g, su, step * 256 + sub0, ("project", step, sub0))
        return p

    ut, uh, up, un = (torch.zeros((n, sm.Wu), dtype=torch.int32, device="cuda") for _ in range(4))
    advect(uw, None, rho, 0, ut)
    pw = projection(ut, pw, 1, uh)
    advect(uh, ut, None, 100, up)
    pw = projection(up, pw, 101, un)
    rho_n = torch.zeros_like(rho)
    sm.advect_density(rho, un, rho_n, dt)
    o = osm.advect(rho.cpu().numpy().astype(np.float64), dec_u(un), dt, dx)
    lo, hi = params["source_lo"], params["source_hi"]
    o[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = 1.0
    check_close(rho_n.cpu().numpy(), o, ("rho", step))
    return un, pw, rho_n


@pytest.mark.parametrize("res,iters,su,steps", [
    ((16, 12, 10), 4, None, 2),
    ((18, 7, 11), 3, None, 1),                          # odd sweep count: the p copy-back
    ((10, 6, 8), 2, schemes.smoke_u_shared(), 1),       # SHARED_EXP velocity (reading Q4)
    ((12, 8, 6), 2, schemes.smoke_u(rounding="rne"), 1),
    ((8, 6, 6), 0, schemes.smoke_raw(6), 1),             # no sweeps, fp32 records
    ((12, 10, 8), 3, "p_shared", 1),                     # SHARED_EXP pressure (reading Q4)
    ((4, 4, 4), 98, None, 1),                            # the largest sweep count (dither subs up to 199)
])
def test_graph_step_equals_checked_chain(res, iters, su, steps):
    sp = None
    if su == "p_shared":
        su, sp = None, schemes.smoke_p_shared()
    params, su, sp, uw, uq, pw, pq, rho = make(res, seed=5, su=su, sp=sp, iters=iters)
    sm = qsmoke.Smoke(params, su, sp)
    sm.set_state(dev(uw), dev(pw), dev(rho), step=3)
    sm.step(steps)
    g_u, g_p, g_rho = sm.get_state_numpy()
    cu, cp, crho = dev(uw), dev(pw), dev(rho)
    for s in range(steps):
        cu, cp, crho = chained_step(sm, params, su, sp, cu, cp, crho, 3 + s, iters)
    assert np.array_equal(g_u, host_u32(cu))
    assert np.array_equal(g_p, host_u32(cp))
    assert np.array_equal(g_rho, crho.cpu().numpy())
    assert sm.launch_count() > 0
    sm.close()


def test_graph_step_against_oracle_step():
    """qsmoke_step against the oracle's own whole step (oracle inputs only): dithering
    decisions may differ where fp32 and fp64 values straddle a threshold, so the decoded
    fields agree to a few quanta (the chained test above is the bit-exact one)."""
    res = (16, 12, 10)
    params, su, sp, uw, uq, pw, pq, rho = make(res, seed=8, iters=8)
    sm = qsmoke.Smoke(params, su, sp)
    sm.set_state(uw, pw, rho, step=0)
    sm.step(1)
    g_u, g_p, g_rho = sm.get_state_numpy()
    o_u, o_p, o_rho = osm.step((uw, pw, rho), params, su, sp, 0, iters=8)
    du = np.abs(osm.decode(g_u, su, res, 3) - osm.decode(o_u, su, res, 3))
    delta_u = su["fields"][0]["range"] * 2.0 ** -su["fields"][0]["frac_bits"]
    assert np.percentile(du, 99) <= 8 * delta_u and du.max() <= 128 * delta_u, (np.percentile(du, 99), du.max())
    assert np.abs(g_rho - o_rho).max() < 1e-2
    sm.close()


def test_errors_are_reported():
    params, _, _, _ = scenes.smoke(res=(8, 8, 8))
    bad = dict(params, res=(7, 8, 8))
    with pytest.raises(qsmoke.qmpm.QmpmError) as e:
        qsmoke.Smoke(bad, schemes.smoke_u(), schemes.smoke_p())
    assert e.value.code == 1
    with pytest.raises(qsmoke.qmpm.QmpmError) as e:
        qsmoke.Smoke(params, schemes.smoke_p(), schemes.smoke_p())
    assert e.value.code == 2


def test_far_departure_points_take_the_global_path():
    """Velocities of several cells per step: most departure points leave the kernels'
    shared-memory window (2 cells), so the global-memory sampling path is the one checked
    against the oracle here (same arithmetic as the window path)."""
    res = (20, 10, 40)
    params, su, sp, uw, uq, pw, pq, rho = make(res, seed=9, su=schemes.smoke_u(rng=16.0), amp=8.0, dt=0.1)
    sm = qsmoke.Smoke(params, su, sp)
    n, dx, dt = sm.n_records, params["dx"], params["dt"]
    assert 8.0 * 0.5 * dt / dx > 2.0  # departures beyond the window
    bdt = 0.5 * dt * params["buoyancy"]
    for refl in (False, True):
        out = torch.zeros((n, sm.Wu), dtype=torch.int32, device="cuda")
        dbg = torch.zeros((n, 6), dtype=torch.float32, device="cuda")
        if refl:
            _, _, _, uw2, uq2, _, _, _ = make(res, seed=10, su=su, amp=8.0, dt=0.1)
            sm.advect_velocity(dev(uw), out, 0.5 * dt, u_refl=dev(uw2), dstep=5 * 256 + 100, dbg=dbg)
            o = osm.sample(2.0 * uq - uq2, osm.backtrace(uq, 0.5 * dt, dx))
            ds = 5 * 256 + 100
        else:
            sm.advect_velocity(dev(uw), out, 0.5 * dt, rho=dev(rho), bdt=bdt, dstep=5 * 256, dbg=dbg)
            o = osm.advect(uq, uq, 0.5 * dt, dx)
            o[..., 1] += bdt * rho.astype(np.float64)
            ds = 5 * 256
        g_pre = dbg.cpu().numpy()
        check_close(g_pre, osm.to_records(o, 3), ("far advect", refl))
        check_words(host_u32(out), g_pre, su, ds, ("far advect", refl))
    outr = torch.zeros(res, dtype=torch.float32, device="cuda")
    sm.advect_density(dev(rho), dev(uw), outr, dt)
    o = osm.advect(rho.astype(np.float64), uq, dt, dx)
    lo, hi = params["source_lo"], params["source_hi"]
    o[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = 1.0
    check_close(outr.cpu().numpy(), o, "far rho")
    sm.close()


@pytest.mark.parametrize("iters", [4, 5])
def test_fused_two_sweep_jacobi_is_bit_identical(iters, monkeypatch):
    """qsmoke_jacobi2 (two sweeps per launch, QSMOKE_FUSE=1; off by default because it is
    slower) against the chain of single sweeps: identical words."""
    monkeypatch.setenv("QSMOKE_FUSE", "1")
    res = (20, 18, 40)  # several y and z tiles of the fused kernel
    params, su, sp, uw, uq, pw, pq, rho = make(res, seed=12, iters=iters)
    sm = qsmoke.Smoke(params, su, sp)
    sm.set_state(dev(uw), dev(pw), dev(rho), step=2)
    sm.step(1)
    g_u, g_p, g_rho = sm.get_state_numpy()
    cu, cp, crho = chained_step(sm, params, su, sp, dev(uw), dev(pw), dev(rho), 2, iters)
    assert np.array_equal(g_u, host_u32(cu)) and np.array_equal(g_p, host_u32(cp))
    assert np.array_equal(g_rho, crho.cpu().numpy())
    sm.close()
