"""Benchmark of the quantized Eulerian smoke step (include/qsmoke.h).

Workload: the paper's large-scale smoke (T-large: 228,982,784 active voxels, dt
0.01, 64 Jacobi iterations per projection) as a dense 612^3 collocated grid
(229,220,928 voxels), velocity 6 x 16-bit and pressure 2 x 16-bit records per two cells
(64 bits per voxel vs 128 in fp32: 2.0x; the paper's scheme: 1.93x).  Scene: a plume
(fluid at rest, density source at the bottom centre, buoyancy), developed for
--scene-warmup steps before the warm-up.  One JSON line like bench.py's.

    python bench_smoke.py [--res 612 612 612] [--steps 5] [--warmup 3]
    python bench_smoke.py --impl reference      # the oracle on a bounded sample

Single GPU only (the smoke path has no slab decomposition yet: DESIGN.md §12).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--res", type=int, nargs=3, default=[612, 612, 612])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--scene-warmup", type=int, default=10)
    ap.add_argument("--iters", type=int, default=64)
    ap.add_argument("--reps", type=int, default=10, help="launches per kernel in the per-kernel timing")
    ap.add_argument("--cpu-res", type=int, nargs=3, default=[64, 64, 64])
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def workload(res, iters):
    n = res[0] * res[1] * res[2]
    return (f"smoke {res[0]}x{res[1]}x{res[2]} ({n:,} voxels; paper T-large: 228,982,784), advection-reflection, "
            f"RK-3 semi-Lagrangian, {iters} Jacobi sweeps x 2 projections, u 6x16-bit + p 2x16-bit records per 2 cells")


def cpu_rate(res, steps, iters):
    """The oracle as it stands (numpy fp64 + the plain-C codec, one thread) on a smaller
    grid of the same scene recipe; returns voxel-steps/s."""
    import numpy as np
    from oracle import smoke as osm
    from paper_2207_04658_b200 import scenes, schemes
    params, u, p, rho = scenes.smoke(res=tuple(res), amp=0.3, jacobi_iters=iters)
    su, sp = schemes.smoke_u(), schemes.smoke_p()
    uw, _ = osm.store(u.astype(np.float64), su, 0, 255, 3)
    pw, _ = osm.store(p[..., None].astype(np.float64), sp, 0, 255, 1)
    state = (uw, pw, rho)
    t0 = time.perf_counter()
    for s in range(steps):
        state = osm.step(state, params, su, sp, s, iters=iters)
    dt = time.perf_counter() - t0
    n = res[0] * res[1] * res[2]
    return n * steps / dt, dt


def run_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    res = args.cpu_res
    n = res[0] * res[1] * res[2]
    rate, secs = cpu_rate(res, max(1, args.steps if args.steps <= 2 else 2), args.iters)
    line = {"impl": "reference", "metric": "quantized smoke voxel-steps/sec", "value": rate, "unit": "voxel-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": n / rate * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args.res, args.iters), "sample": f"{res} grid"},
            "cpu_baseline": {"value": rate, "unit": "voxel-steps/s", "cores": 1, "kind": "oracle",
                             "sample": f"{res[0]}x{res[1]}x{res[2]} grid of the same recipe ({secs:.1f} s)"},
            "e2e": {"value": rate, "unit": "voxel-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_gpu(args):
    import torch
    from bench import ClockSampler
    from paper_2207_04658_b200 import qsmoke, scenes, schemes

    torch.cuda.set_device(0)
    res = tuple(args.res)
    nvox = res[0] * res[1] * res[2]
    params = scenes.smoke_plume(res, jacobi_iters=args.iters)
    su, sp = schemes.smoke_u(), schemes.smoke_p()
    stream = torch.cuda.current_stream()
    sm = qsmoke.Smoke(params, su, sp, stream=stream)
    n = sm.n_records
    u = torch.zeros((n, sm.Wu), dtype=torch.int32, device="cuda")
    p = torch.zeros((n, sm.Wp), dtype=torch.int32, device="cuda")
    rho = torch.zeros(res, dtype=torch.float32, device="cuda")
    sm.set_state(u, p, rho)
    sm.step(args.scene_warmup + args.warmup)
    torch.cuda.synchronize()

    # ---------------- timed region: K steps (CUDA graph replays) on the ctx stream
    launches0 = sm.launch_count()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sm.step(args.steps)
    e1.record(stream)
    e1.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    launches = sm.launch_count() - launches0
    value = nvox * args.steps / (ms / 1e3)

    # ---------------- per-kernel times (events around `reps` launches of each sub-step
    # kernel on the current state, same stream): the shares of the step
    sm.get_state(u, p, rho)
    u2, p2 = torch.empty_like(u), torch.empty_like(p)
    div = torch.empty(res, dtype=torch.float32, device="cuda")
    rho2 = torch.empty_like(rho)
    dt = params["dt"]
    sm.divergence(u, div)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.reps):
            fn()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b) / args.reps

    kms = {"advect_velocity": timed(lambda: sm.advect_velocity(u, u2, 0.5 * dt, rho=rho, bdt=0.005, dstep=1)),
           "advect_reflect": timed(lambda: sm.advect_velocity(u, u2, 0.5 * dt, u_refl=u, dstep=1)),
           "divergence": timed(lambda: sm.divergence(u, div)),
           "jacobi": timed(lambda: sm.jacobi(p, div, p2, dstep=2)),
           "project": timed(lambda: sm.project(u, p, u2, dstep=3)),
           "advect_density": timed(lambda: sm.advect_density(rho, u, rho2, dt))}
    per_step = {"advect_velocity": 1, "advect_reflect": 1, "divergence": 2, "jacobi": 2 * args.iters, "project": 2,
                "advect_density": 1}
    shares = {k: {"ms_per_launch": v, "launches_per_step": per_step[k], "ms_per_step": v * per_step[k],
                  "share_of_step": v * per_step[k] / (ms / args.steps)} for k, v in kms.items()}
    del u2, p2, rho2

    # ---------------- roofline of the dominant kernel (Jacobi: HBM-bound stencil)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        hbm_peak, src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        hbm_peak, src = 6650.0, "fallback (B200_PROFILING.md)"
    dom = max(shares, key=lambda k: shares[k]["ms_per_step"])
    alg = {"jacobi": n * (2 * 4 * sm.Wp + 8),             # p read + p written + 2 fp32 div per record
           "project": n * (2 * 4 * sm.Wu + 4 * sm.Wp),
           "divergence": n * (4 * sm.Wu + 8),
           "advect_velocity": n * (2 * 4 * sm.Wu + 8),
           "advect_reflect": n * (3 * 4 * sm.Wu),
           "advect_density": n * (4 * sm.Wu + 16)}[dom]
    achieved = alg / (kms[dom] / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic_smoke.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic, "peak_source": src,
                "algorithmic_bytes_per_launch": alg, "avg_launch_ms": kms[dom],
                "timing": "events around back-to-back launches of that kernel alone (the step is one CUDA graph)"}

    # ---------------- end to end through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        hu = torch.empty((n, sm.Wu), dtype=torch.int32, pin_memory=True)
        hp = torch.empty((n, sm.Wp), dtype=torch.int32, pin_memory=True)
        hr = torch.empty(res, dtype=torch.float32, pin_memory=True)
        sm.get_state(hu, hp, hr)
        k = args.steps
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sm.set_state(hu, hp, hr, step=100)   # H2D of the state (pinned)
        sm.step(k)
        sm.get_state(hu, hp, hr)             # D2H of the result (synchronizes)
        e2e_s = time.perf_counter() - t0
        nb = n * 4 * (sm.Wu + sm.Wp) + 4 * nvox
        e2e = {"value": nvox * k / e2e_s, "unit": "voxel-steps/s", "h2d_bytes_per_step": int(nb / k),
               "d2h_bytes_per_step": int(nb / k),
               "note": f"timed: qsmoke_set_state(pinned host, {nb / 1e9:.2f} GB) + {k} x qsmoke_step + "
                       "qsmoke_get_state(-> pinned host)"}
    sm.close()

    cpu = None
    if not args.no_cpu:
        rate, secs = cpu_rate(args.cpu_res, args.cpu_steps, args.iters)
        cr = args.cpu_res
        cpu = {"value": rate, "unit": "voxel-steps/s", "cores": 1, "kind": "oracle",
               "sample": f"{cr[0]}x{cr[1]}x{cr[2]} grid of the same recipe, {args.cpu_steps} step(s) "
                         f"(numpy fp64 + plain-C codec, 1 thread, {secs:.1f} s)"}

    bits = 32 * (sm.Wu + sm.Wp) / 2
    line = {
        "metric": "quantized smoke voxel-steps/sec", "value": value, "unit": "voxel-steps/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload(res, args.iters), "voxels": nvox, "bits_per_voxel": bits,
                   "compression_vs_fp32": 128.0 / bits, "scene_warmup_steps": args.scene_warmup,
                   "l2": f"state {n * 4 * (sm.Wu + sm.Wp) / 1e9:.2f} GB + div {4 * nvox / 1e9:.2f} GB >> 126 MB L2",
                   "parallelism": "single GPU"},
        "roofline": roofline,
        "kernels": shares,
        "gpu_launches": int(launches),
        "e2e": e2e,
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
