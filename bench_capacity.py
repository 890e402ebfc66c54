"""Capacity probe: the largest particle count one B200 holds for the
fp32 layout vs a quantized scheme, with the SAME code and every per-particle array
counted (two record buffers, sort key, permutation), at the C3 grid.

    python bench_capacity.py [--schemes fp32,e0.01] [--grid 1024]

For each scheme it bisects max_particles for which qmpm_create succeeds AND one step
runs (a compact lattice of that many particles), then prints one JSON line with the
capacities, their ratio and the analytic bytes per particle.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def try_n(sc_fn, sch, n, torch, qmpm):
    sc = sc_fn(n)
    try:
        sim = qmpm.Sim(sc.sim, sch, n, flags=qmpm.NO_ROUND_COUNTERS)
    except qmpm.QmpmError:
        return False
    try:
        chunk = 1 << 24
        for s0 in range(0, n, chunk):
            st = sc.state_chunk(s0, min(chunk, n - s0), backend="torch", device="cuda")
            (sim.set_state if s0 == 0 else sim.append_state)(st)
            torch.cuda.synchronize()
            del st
        torch.cuda.empty_cache()
        sim.step(1)
        torch.cuda.synchronize()
        ok = sim.stats().n_particles == n
    except Exception:
        ok = False
    sim.close()
    torch.cuda.empty_cache()
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--schemes", default="fp32,e0.01")
    ap.add_argument("--lo", type=float, default=1e8)
    ap.add_argument("--tol", type=float, default=0.02)
    args = ap.parse_args()
    import torch
    from paper_2207_04658_b200 import qmpm, scenes, schemes
    torch.cuda.set_device(0)
    free, total = torch.cuda.mem_get_info()

    def scene(n):
        # elastic cubes on the 1024^3 grid (C3's layout, more cubes as n grows)
        return scenes.c3(n_target=n, cube=209)

    out = {"gpu_total_bytes": total, "gpu_free_bytes": free, "grid": 1024, "capacity": {}, "bytes_per_particle": {}}
    for name in args.schemes.split(","):
        sch = schemes.fp32(3) if name == "fp32" else schemes.BY_NAME[name]()
        _, W, _ = qmpm.layout(sch)
        out["bytes_per_particle"][name] = 2 * 4 * W + 4 + 4  # records x2, key, perm
        lo = int(args.lo)
        if not try_n(scene, sch, lo, torch, qmpm):
            out["capacity"][name] = None
            continue
        hi = lo * 2
        while try_n(scene, sch, min(hi, scenes.C3_PARTICLES * 6), torch, qmpm) and hi < scenes.C3_PARTICLES * 6:
            lo, hi = hi, hi * 2
        while hi - lo > args.tol * lo:
            mid = (lo + hi) // 2
            if try_n(scene, sch, mid, torch, qmpm):
                lo = mid
            else:
                hi = mid
        out["capacity"][name] = lo
    caps = out["capacity"]
    names = args.schemes.split(",")
    if len(names) >= 2 and caps.get(names[0]) and caps.get(names[1]):
        out["ratio"] = caps[names[1]] / caps[names[0]]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
