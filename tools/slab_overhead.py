"""Per-step overhead of the slab decomposition, measured on ONE GPU with the in-process
group transport (qmpm_step_group): the C4 scene (n particles) as one context vs k z slabs
stepping together.  The slab path adds the leaver routing in G2P, the device-side
append of arrivals, the ghost / velocity plane packs and the split P2G / G2P launches
(no host synchronisation per step since round 2); with k slabs on one GPU their
kernels and exchange copies run back to back on one stream, so (t_k - t_1) / k
estimates the per-rank overhead of an N-GPU weak-scaling step (the NCCL transfers
themselves are not in it).

    python tools/slab_overhead.py [--n 200000000] [--k 2] [--steps 10]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200_000_000)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warm", type=int, default=20)
    ap.add_argument("--weak", action="store_true",
                    help="the decomposition bench.py --gpus k uses: --n particles PER SLAB, the C4 scene "
                         "extended k times along z (one 256^3 slab per rank); skips the single-ctx run")
    args = ap.parse_args()
    import torch
    from paper_2207_04658_b200 import dist as qdist
    from paper_2207_04658_b200 import qmpm, scenes, schemes
    torch.cuda.set_device(0)
    if args.weak:
        sc = scenes.c4(n_target=args.n * args.k, z_extent=float(args.k))
        sch = schemes.with_domain(schemes.f2(), sc.sim)  # (x_z over [0, k), as bench.py)
    else:
        sc, sch = scenes.c4(n_target=args.n), schemes.f2()
    stream = torch.cuda.Stream()
    out = {"n": sc.n_particles, "k": args.k, "weak": args.weak}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        if not args.weak:
            sim = qmpm.Sim(sc.sim, sch, sc.n_particles, stream=stream)
            chunk = 1 << 24
            for s0 in range(0, sc.n_particles, chunk):
                st = sc.state_chunk(s0, min(chunk, sc.n_particles - s0), backend="torch", device="cuda")
                (sim.set_state if s0 == 0 else sim.append_state)(st)
                stream.synchronize()
            sim.step(args.warm)
            stream.synchronize()
            e0.record(stream)
            sim.step(args.steps)
            e1.record(stream)
            e1.synchronize()
            out["single_ms"] = e0.elapsed_time(e1) / args.steps
            sim.close()
            torch.cuda.empty_cache()
        cuts = qdist.slab_cuts(sc.sim["grid_res"][2], args.k)
        sims = []
        for r in range(args.k):
            s = qmpm.Sim(sc.sim, sch, qdist.slab_capacity(sc, cuts, r), stream=stream,
                         slab=(args.k, r, cuts[r][0], cuts[r][1]))  # (capacities reconciled by the group)
            qdist.load_slab(s, sc, cuts, r, track_ids=False)
            sims.append(s)
        qmpm.step_group(sims, args.warm)
        stream.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        qmpm.step_group(sims, args.steps)
        e1.record(stream)
        e1.synchronize()
        out["group_ms"] = e0.elapsed_time(e1) / args.steps
        out["group_wall_ms"] = (time.perf_counter() - t0) * 1e3 / args.steps
        if "single_ms" in out:
            out["overhead_per_slab_ms"] = (out["group_ms"] - out["single_ms"]) / args.k
        out["n_per_slab"] = [s.stats().n_particles for s in sims]
        # per-kernel device time of the group step (events around every launch), summed
        # over the slabs, ms per step -- where the extra time of a slab step goes
        for s in sims:
            s.set_profiling(True)
        qmpm.step_group(sims, args.steps)
        stream.synchronize()
        kt = {}
        for s in sims:
            for name, (ms, cnt) in s.kernel_times().items():
                if cnt:
                    kt[name] = kt.get(name, 0.0) + ms / args.steps
            s.set_profiling(False)
        out["group_kernel_ms_per_step"] = {k: round(v, 3) for k, v in sorted(kt.items(), key=lambda x: -x[1])}
        for s in sims:
            s.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
