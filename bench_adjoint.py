"""Benchmark of the gradient tallies (Algorithm 1 line 12; SURVEY §8(f) row f3;
include/qadjoint.h): T forward fp32 steps, KE(s_T), back-propagation with the paper's
bisection checkpointing, g_h per state scalar.

Default workload: the paper's error-bounded MPM experiment (an elastic body,
80,000 particles, 128^2 grid, 8192 steps, dt 2e-4): 2D fixed-corotated, 283^2 = 80,089
particles at 16 per cell.  --config 3d: 1M elastic particles (100^3, 8 per cell) on
128^3, T = 64; 2d-fluid / 3d-fluid: the same with the J-fluid.

    python bench_adjoint.py [--config 2d|3d|2d-fluid|3d-fluid] [--steps T]
    python bench_adjoint.py --impl reference     # the numpy oracle on a bounded sample

One JSON line: metric = particle-steps of the whole tally (n T) per second.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {"2d": dict(material="elastic", dim=2, side=283, res=128, ppc=4, T=8192, origin=0.2),
           "3d": dict(material="elastic", dim=3, side=100, res=128, ppc=2, T=64, origin=0.2),
           "2d-fluid": dict(material="fluid", dim=2, side=283, res=128, ppc=4, T=8192, origin=0.2),
           "3d-fluid": dict(material="fluid", dim=3, side=100, res=128, ppc=2, T=64, origin=0.2)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", default="2d", choices=list(CONFIGS))
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="T (default: the config's)")
    ap.add_argument("--warmup", type=int, default=3, help="warm-up tallies with T = 4")
    ap.add_argument("--cpu-steps", type=int, default=8)
    ap.add_argument("--repeats", type=int, default=3, help="timed tallies (the median is reported)")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def scene(cfg):
    from paper_2207_04658_b200 import scenes
    kw = dict(dim=cfg["dim"], side=cfg["side"], res=cfg["res"], ppc=cfg["ppc"], seed=0, vmax=0.5, cmax=0.5,
              origin=cfg["origin"])
    if cfg["material"] == "fluid":
        return scenes.adjoint_fluid(dJ=0.01, **kw)
    return scenes.adjoint_elastic(dF=0.01, **kw)


def workload(cfg, n, T):
    mat = "J-fluid" if cfg["material"] == "fluid" else "fixed-corotated elastic"
    return (f"gradient tallies, {cfg['dim']}D {mat}, {n:,} particles, {cfg['res']}^{cfg['dim']} grid, T = {T} "
            f"steps, KE(s_T), bisection checkpointing")


def cpu_rate(cfg, steps):
    """The oracle as it stands (numpy fp64 + the C forward, store-all, one thread)."""
    from oracle import adjoint as adj
    sim, s0 = scene(cfg)
    t0 = time.perf_counter()
    adj.backward_all(sim, s0, steps)
    dt = time.perf_counter() - t0
    return s0.shape[0] * steps / dt, dt, s0.shape[0]


def run_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cfg = CONFIGS[args.config]
    T = args.steps or cfg["T"]
    rate, secs, n = cpu_rate(cfg, args.cpu_steps)
    line = {"impl": "reference", "metric": "gradient-tally particle-steps/sec", "value": rate,
            "unit": "particle-steps/s", "n_gpus": args.gpus, "steps": T, "warmup": args.warmup,
            "ms_per_step": n / rate * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": {"workload": workload(cfg, n, T)},
            "cpu_baseline": {"value": rate, "unit": "particle-steps/s", "cores": 1, "kind": "oracle",
                             "sample": f"T = {args.cpu_steps} store-all ({secs:.1f} s)"},
            "e2e": {"value": rate, "unit": "particle-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_gpu(args):
    import torch
    from bench import ClockSampler
    from paper_2207_04658_b200 import qadjoint

    torch.cuda.set_device(0)
    cfg = CONFIGS[args.config]
    T = args.steps or cfg["T"]
    sim, s0 = scene(cfg)
    n, ns = s0.shape
    stream = torch.cuda.current_stream()
    A = qadjoint.Adjoint(sim, n, stream=stream)
    s0d = torch.from_numpy(s0).cuda()
    for _ in range(args.warmup):
        A.gradient_tally(s0d, 4)
    torch.cuda.synchronize()
    l0 = A.launch_count()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    times = []
    for _ in range(args.repeats):  # the median of `repeats` whole tallies
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g, z, st = A.gradient_tally(s0d, T)  # synchronizes
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    clk = clocks.stop()
    ms = sorted(times)[len(times) // 2]
    launches = (A.launch_count() - l0) // args.repeats
    # e2e: the initial state from pinned host memory, tallies back to the host
    hs = torch.from_numpy(s0).pin_memory()
    t0 = time.perf_counter()
    A.gradient_tally(hs, T)
    e2e_s = time.perf_counter() - t0
    # per-kernel split: one forward and one adjoint step, events around each
    so = torch.empty_like(s0d)
    lam = torch.zeros_like(s0d)
    lam2 = torch.empty_like(s0d)

    def timed(fn, reps=20):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b) / reps

    f_ms = timed(lambda: A.forward(s0d, so))
    a_ms = timed(lambda: A.adjoint_step(s0d, lam, lam2))
    nn = 1
    for a in range(cfg["dim"]):
        nn *= cfg["res"]
    A.close()
    # roofline of the adjoint step (5 kernels): algorithmic bytes = the state rows it must
    # read / write (s twice, lambda_{t+1}, lambda_t written and re-read, the fx partials)
    # plus each dense-grid pass (16 B per node: P2G write, grid read + gv write + lgrid
    # clear, node-adjoint scatter, grid-adjoint read 2 + write 1 + clear 1, P2G-adjoint
    # gather)
    row = 4 * ns
    alg = n * (2 * row + row + 2 * row + 2 * 12) + nn * 16 * 10
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm_peak = float(json.load(open(peaks_path))["hbm_gbs"]) if os.path.exists(peaks_path) else 6650.0
    achieved = alg / (a_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": "adjoint step (5 kernels)", "achieved": achieved, "peak": hbm_peak,
                "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": None,
                "algorithmic_bytes_per_launch": alg, "avg_launch_ms": a_ms,
                "note": "small scenes are bound by P2G / node-adjoint atomics, not bytes (DESIGN.md §13)"}
    value = n * T / (ms / 1e3)
    cpu = None
    if not args.no_cpu:
        rate, secs, _ = cpu_rate(cfg, args.cpu_steps)
        cpu = {"value": rate, "unit": "particle-steps/s", "cores": 1, "kind": "oracle",
               "sample": f"the same scene, T = {args.cpu_steps}, store-all (numpy fp64 + C forward, 1 thread, "
                         f"{secs:.1f} s)"}
    line = {
        "metric": "gradient-tally particle-steps/sec", "value": value, "unit": "particle-steps/s", "n_gpus": 1,
        "steps": T, "warmup": args.warmup, "ms_per_step": ms / T, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload(cfg, n, T), "particles": n, "state_bytes": n * ns * 4,
                   "parallelism": "single GPU"},
        "timed_tallies_ms": times,
        "checkpointing": {"max_resident_states": st["max_resident"], "forward_steps": st["forward_steps"],
                          "adjoint_steps": st["adjoint_steps"], "log2_T": math.log2(max(T, 1))},
        "roofline": roofline,
        "kernels": {"forward_step_ms": f_ms, "adjoint_step_ms": a_ms,
                    "model_ms": st["forward_steps"] * f_ms + st["adjoint_steps"] * a_ms},
        "z": z, "g": g.tolist(),
        "gpu_launches": int(launches),
        "e2e": {"value": n * T / e2e_s, "unit": "particle-steps/s", "h2d_bytes_per_step": int(n * ns * 4 / T),
                "d2h_bytes_per_step": int(8 * (ns + 1) / T), "note": "s0 from pinned host, g and z back to the host"},
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
