"""Per-kernel timing of the smoke step at a given resolution (development probe).

    python tools/smoke_probe.py [--res 612 612 612] [--steps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--res", type=int, nargs=3, default=[612, 612, 612])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ncu", action="store_true", help="after 4 plume steps (540 launches) run each sub-step kernel once")
    a = ap.parse_args()
    import torch
    from paper_2207_04658_b200 import qsmoke, scenes, schemes
    params = scenes.smoke_plume(tuple(a.res))
    su, sp = schemes.smoke_u(), schemes.smoke_p()
    sm = qsmoke.Smoke(params, su, sp)
    n = sm.n_records
    nc = 2 * n
    st = torch.cuda.current_stream()
    u = torch.zeros((n, sm.Wu), dtype=torch.int32, device="cuda")
    p = torch.zeros((n, sm.Wp), dtype=torch.int32, device="cuda")
    rho = torch.zeros(tuple(a.res), dtype=torch.float32, device="cuda")
    sm.set_state(u, p, rho)
    sm.step(4)  # develop the plume a little
    torch.cuda.synchronize()

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    if a.ncu:
        sm.get_state(u, p, rho)
        u2, p2 = torch.empty_like(u), torch.empty_like(p)
        div = torch.zeros(tuple(a.res), dtype=torch.float32, device="cuda")
        rho2 = torch.empty_like(rho)
        dt = params["dt"]
        sm.advect_velocity(u, u2, 0.5 * dt, rho=rho, bdt=0.005, dstep=1)
        sm.advect_velocity(u, u2, 0.5 * dt, u_refl=u, dstep=1)
        sm.divergence(u, div)
        sm.jacobi(p, div, p2, dstep=2)
        sm.project(u, p, u2, dstep=3)
        sm.advect_density(rho, u, rho2, dt)
        torch.cuda.synchronize()
        print("ncu pass done", flush=True)
        return
    out = {"res": a.res, "records": n, "Wu": sm.Wu, "Wp": sm.Wp}
    out["step_ms"] = timed(lambda: sm.step(1), a.steps)
    sm.get_state(u, p, rho)
    u2, p2 = torch.empty_like(u), torch.empty_like(p)
    div = torch.zeros(tuple(a.res), dtype=torch.float32, device="cuda")
    rho2 = torch.empty_like(rho)
    dt = params["dt"]
    out["advect_u_ms"] = timed(lambda: sm.advect_velocity(u, u2, 0.5 * dt, rho=rho, bdt=0.005, dstep=1), a.reps)
    out["advect_refl_ms"] = timed(lambda: sm.advect_velocity(u, u2, 0.5 * dt, u_refl=u, dstep=1), a.reps)
    out["div_ms"] = timed(lambda: sm.divergence(u, div), a.reps)
    out["jacobi_ms"] = timed(lambda: sm.jacobi(p, div, p2, dstep=2), a.reps)
    out["project_ms"] = timed(lambda: sm.project(u, p, u2, dstep=3), a.reps)
    out["advect_rho_ms"] = timed(lambda: sm.advect_density(rho, u, rho2, dt), a.reps)
    jb = n * (2 * 4 * sm.Wp + 8)
    out["jacobi_GBps"] = jb / out["jacobi_ms"] / 1e6
    out["voxel_steps_per_s"] = nc / out["step_ms"] * 1e3
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
