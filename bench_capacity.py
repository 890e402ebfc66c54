"""Capacity probe (BASELINE north_star: "holding >= 2x more particles
per GPU than fp32 at the paper's 0.01 error bound"): the largest particle count one
B200 holds for the fp32 layout vs a quantized scheme, with the SAME code and every
device array counted, on C3's 1024^3 grid.

    python bench_capacity.py [--schemes fp32,e0.01]

Per scheme: bytes per particle = two record buffers (2 x 4W) + sort key (4) + perm (4)
+ the grid pool share of an 8-ppc block (64-node blocks, 1 per 512 particles, x 1.25
for touched neighbours, 2 float4 arrays); fixed = cell counters (64 x 4 B per grid
block) + block tables.  The prediction N = (free - fixed - margin) / bytes is then
VERIFIED: a Sim of max_particles = N is created, filled with a dense elastic block of
N particles (scenes.dense_elastic) and stepped twice; on failure N shrinks by 3 %.
One JSON line: capacities, their ratio and the byte accounting.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GRID = 1024
NBLOCKS = (GRID // 4) ** 3


def grid_bytes_per_particle():
    return 1.25 * 2 * 64 * 16 / 512  # touched blocks per particle x 2 float4 arrays


def try_n(n, sch, torch, qmpm, scenes):
    sc = scenes.dense_elastic(n, GRID)
    pool = int(1.25 * n / 512) + 4096
    sim = None
    try:
        sim = qmpm.Sim(sc.sim, sch, n, flags=qmpm.NO_ROUND_COUNTERS, pool_blocks=pool)
        chunk = 1 << 24
        for s0 in range(0, n, chunk):
            st = sc.state_chunk(s0, min(chunk, n - s0), backend="torch", device="cuda")
            (sim.set_state if s0 == 0 else sim.append_state)(st)
            torch.cuda.synchronize()
            del st
        torch.cuda.empty_cache()
        sim.step(2)
        st = sim.stats()
        ok = st.n_particles == n and st.pool_overflow == 0
    except Exception as e:  # allocation failure (qmpm ENOMEM or torch OOM)
        print(f"  n={n}: {type(e).__name__}: {str(e)[:120]}", file=sys.stderr)
        ok = False
    if sim is not None:
        sim.close()
    torch.cuda.empty_cache()
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--schemes", default="fp32,e0.01")
    ap.add_argument("--margin-gb", type=float, default=3.0)
    args = ap.parse_args()
    import torch
    from paper_2207_04658_b200 import qmpm, scenes, schemes
    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")
    free, total = torch.cuda.mem_get_info()
    fixed = NBLOCKS * (64 * 4 + 4 * 4 + 4)  # cell counters + block tables (+ scan scratch)
    out = {"gpu_total_bytes": total, "gpu_free_bytes": free, "grid": GRID, "fixed_bytes": fixed,
           "capacity": {}, "bytes_per_particle": {}, "predicted": {}, "tries": {}}
    for name in args.schemes.split(","):
        sch = schemes.fp32(3) if name == "fp32" else schemes.BY_NAME[name]()
        _, W, _ = qmpm.layout(sch)
        bpp = 2 * 4 * W + 4 + 4 + grid_bytes_per_particle()
        out["bytes_per_particle"][name] = bpp
        n = int((free - fixed - args.margin_gb * 1e9) / bpp)
        out["predicted"][name] = n
        cap = None
        for t in range(4):
            print(f"{name}: trying n={n}", file=sys.stderr, flush=True)
            if try_n(n, sch, torch, qmpm, scenes):
                cap = n
                break
            n = int(n * 0.97)
        out["capacity"][name] = cap
        out["tries"][name] = t + 1
    caps = out["capacity"]
    names = args.schemes.split(",")
    if len(names) >= 2 and caps.get(names[0]) and caps.get(names[1]):
        out["ratio"] = caps[names[1]] / caps[names[0]]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
