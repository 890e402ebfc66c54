"""bench.py -- quantized MLS-MPM particle-steps/s and % HBM roofline on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--scheme e0.01]
    python bench.py --impl reference ...   (the CPU oracle as it stands, host cores)

Default workload (BASELINE.json configs[3], the paper's T-large fluid run, P:946;
the config its metric is quoted on at 1/2/4/8 GPUs): C4 = 3D fluid dam-break,
400M particles PER GPU (weak scaling: the domain is extended along z by N and cut
into z slabs, one per rank, exchanging ghost planes and migrants over NCCL), 256^3
cells per GPU, dt 1e-4, stand-in scheme F2 (253 bits, W = 8 words).
`--config c3` runs configs[2] instead (295M elastic particles on 1024^3, E0.01,
single GPU).  Inputs are generated on the device (seeded), encoded by
qmpm_set_state, advanced `scene_warmup` untimed steps (so C != 0 and the flow
develops), then W warm-up steps, then K timed steps.  The state (>12 GB) is far
larger than L2 (126 MB), so no flush is needed between steps.

One JSON line on rank 0 (see the contract in the task statement); the roofline
object is for the dominant kernel, with algorithmic bytes per launch defined in
DESIGN.md §6, duration from CUDA events on the ctx stream over the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the OpenMP oracle (cpu_baseline, --impl reference) shares torch's libgomp: passive
# waiting keeps the two thread pools from spinning against each other (read at init)
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

PAPER_PSTEPS = {"c3": 295_280_208 * 128 / 63.5,   # derived from T-large, RTX 3090: context
                "c4": 400_000_000 * 128 / 139.3}   # derived from T-large, RTX 3090: context


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="qmpm", choices=["qmpm", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c4_8ppc"],
                    help="c4_8ppc: C4's 400M particles on 512^3 cells per GPU (~8 ppc, dt 5e-5; SURVEY Q16)")
    ap.add_argument("--scheme", default=None, help="x16 | e0.1 | e0.01 | f2 | fp32")
    ap.add_argument("--n", type=int, default=0, help="override particle count (reduced runs)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="C4 with N > 1 GPUs: weak = 400M per GPU on a z-extended domain (default); "
                         "strong = 400M in total on the 256^3 domain, cut into N z slabs")
    ap.add_argument("--z-extent", type=float, default=1.0,
                    help="C4 only: z extent of the 1-GPU domain (reduced same-density runs for profiling)")
    ap.add_argument("--scene-warmup", type=int, default=None,
                    help="untimed steps before the warm-up so the flow is developed (default: C4 2000 -- the dam "
                         "has started to collapse -- C3 1000 -- the cubes collide --, C1/C2 100)")
    ap.add_argument("--rounding", default="dither", choices=["dither", "rne"])
    ap.add_argument("--layout", default="pack", choices=["pack", "nostraddle"],
                    help="bit pack (P:542-549) or no field straddling a word (the bit struct's rule, P:540)")
    ap.add_argument("--no-counters", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1_000_000)
    ap.add_argument("--cpu-steps", type=int, default=5)
    ap.add_argument("--ref-sample", type=int, default=250_000, help="particles per --impl reference step")
    return ap.parse_args()


def make_scene(args, world=1):
    from paper_2207_04658_b200 import scenes, schemes
    if args.config == "c1":
        sc = scenes.c1()
        sch = schemes.x16()
    elif args.config == "c2":
        sc = scenes.c2()
        sch = schemes.e01()
    elif args.config == "c3":
        sc = scenes.c3(n_target=args.n or scenes.C3_PARTICLES)
        sch = schemes.e001()
    else:
        wx = world if args.scaling == "weak" else 1
        if args.config == "c4_8ppc":
            sc = scenes.c4(n_target=(args.n or 400_000_000) * wx, res=512, dt=5e-5, z_extent=float(wx) * args.z_extent)
            sc.name = "C4-8ppc"
        else:
            sc = scenes.c4(n_target=(args.n or 400_000_000) * wx, z_extent=float(wx) * args.z_extent)
        sch = schemes.f2()
    if args.scheme:
        sch = schemes.fp32(sc.dim, sc.material) if args.scheme == "fp32" else schemes.BY_NAME[args.scheme]()
    # positions over the whole domain (the weak-scaling runs extend C4 along z; a no-op at N = 1)
    sch = schemes.with_domain(sch, sc.sim)
    sch = schemes.with_layout(schemes.with_rounding(sch, args.rounding), args.layout)
    return sc, sch


def scheme_name(args):
    return args.scheme or {"c1": "x16", "c2": "e0.1", "c3": "e0.01", "c4": "f2", "c4_8ppc": "f2"}[args.config]


DEFAULT_SCENE_WARMUP = {"c1": 100, "c2": 100, "c3": 1000, "c4": 2000, "c4_8ppc": 2000}


def workload_name(args, sc, W, bits):
    return (f"{sc.name}: {sc.dim}D {sc.material}, {sc.n_particles:,} particles, "
            f"{'x'.join(str(r) for r in sc.sim['grid_res'][:sc.dim])} block-sparse grid, "
            f"dt {sc.sim['dt']:g}, scheme {scheme_name(args)} ({bits} bits, W={W}"
            + (", no-straddle layout" if args.layout == "nostraddle" else "") + ")")


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- CPU oracle
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_rate(sc, sch, n_sample, steps, threads=1):
    """The oracle (plain C, fp64) on the first n_sample particles of the same workload:
    threads = 1 the single-threaded oracle_step, else its OpenMP particle loops
    (SURVEY §8(d) M7 ii; 0 = all host cores).  Returns (p-steps/s, n, steps, s, threads)."""
    import oracle
    n = min(n_sample, sc.n_particles)
    st = sc.state_chunk(0, n)
    w, _ = oracle.encode_state(sch, st)
    used = 1 if threads == 1 else (oracle.num_threads() if threads <= 0 else threads)
    t0 = time.perf_counter()
    oracle.run(sc.sim, sch, w, 1, steps, threads=threads)
    dt = time.perf_counter() - t0
    return n * steps / dt, n, steps, dt, used


def run_reference(args):
    """The oracle as it stands on the box's host cores (its OpenMP particle loops on all
    cores), on a bounded sample of the same workload per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sc, sch = make_scene(args)
    import oracle
    _, W, bits = oracle.layout(sch)
    n = min(args.ref_sample, sc.n_particles)
    st = sc.state_chunk(0, n)
    w, _ = oracle.encode_state(sch, st)
    cores = oracle.num_threads()
    for t in range(args.warmup):
        w = oracle.step(sc.sim, sch, w, t + 1, threads=0)[1]
    times = []
    for t in range(args.steps):
        t0 = time.perf_counter()
        w = oracle.step(sc.sim, sch, w, args.warmup + t + 1, threads=0)[1]
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = n * args.steps / total
    line = {
        "impl": "reference", "metric": "quantized MPM particle-steps/sec", "value": value,
        "unit": "particle-steps/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args, sc, W, bits), "sample_particles": n},
        "cpu_baseline": {"value": value, "unit": "particle-steps/s", "cores": cores, "kind": "oracle",
                         "sample": f"first {n:,} particles of the workload, {args.steps} steps "
                                   f"(fp64 plain C, OpenMP particle loops on {cores} threads)",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "particle-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU
def algorithmic_bytes(S, nodes):
    """Per launch: P2G reads each record once and reduces 16 B per
    touched node; G2P reads + writes each record and reads 12 B per touched node."""
    return {"p2g": lambda n: n * S + 16 * nodes, "g2p": lambda n: 2 * n * S + 12 * nodes,
            "grid_update": lambda n: 28 * nodes}


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2207_04658_b200 import qmpm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sc, sch = make_scene(args, world)
    _, W, bits = qmpm.layout(sch)
    flags = qmpm.NO_ROUND_COUNTERS if args.no_counters else 0
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        if world == 1:
            N = sc.n_particles
            sim = qmpm.Sim(sc.sim, sch, N, flags=flags, stream=stream)
            chunk = 1 << 24
            for s0 in range(0, N, chunk):
                cnt = min(chunk, N - s0)
                st = sc.state_chunk(s0, cnt, backend="torch", device="cuda")
                if s0 == 0:
                    sim.set_state(st)
                else:
                    sim.append_state(st)
                stream.synchronize()
                del st
        else:
            # slab decomposition along z (one slab per rank), NCCL exchanges
            from paper_2207_04658_b200 import dist as qdist
            if sc.dim != 3:
                raise SystemExit("multi-GPU runs need a 3D config")
            cuts = qdist.slab_cuts(sc.sim["grid_res"][2], world)
            cap = qdist.slab_capacity(sc, cuts, rank)
            sim = qmpm.Sim(sc.sim, sch, cap, flags=flags, stream=stream,
                           slab=(world, rank, cuts[rank][0], cuts[rank][1]))
            uid = qdist.share_unique_id(qmpm.get_unique_id)
            sim.connect_nccl(uid)
            qdist.load_slab(sim, sc, cuts, rank, track_ids=False)
        torch.cuda.empty_cache()
        sim.step(args.scene_warmup + args.warmup)
        stream.synchronize()
        cap = sim.params.max_particles  # this rank's context capacity (host buffers below)

        # ---------------- timed region (device): K steps, per-kernel events on the ctx stream
        # (the step as the library runs it: one CUDA graph per step on a single GPU; the
        # per-kernel event brackets of the roofline are taken in a second pass below)
        launches0 = sim.launch_count()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(local)
        clocks.start()
        time.sleep(0.3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.step(args.steps)
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        clk = clocks.stop()
        launches = sim.launch_count() - launches0
        ms = e0.elapsed_time(e1)
        # ---------------- per-kernel device times (CUDA events around each launch, same stream)
        sim.set_profiling(True)
        sim.step(args.steps)
        ktimes = sim.kernel_times()
        sim.set_profiling(False)
        st = sim.stats()
        N = int(st.n_particles)  # this rank's particles (slabs: after migration)
        n_total = N
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            c = torch.tensor([N], device="cuda", dtype=torch.int64)
            dist.all_reduce(c)
            n_total = int(c.item())
        value = n_total * args.steps / (ms / 1e3)

        # ---------------- end to end through the C ABI with pinned host buffers
        e2e = None
        if not args.no_e2e:
            # sized at the context capacity: a slab's count changes with migration
            host = torch.empty((cap, W), dtype=torch.int32, pin_memory=True)
            n0 = sim.read_state(words=host)  # the current state, as a user would hold it on the host
            step0 = st.step
            k = args.steps
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            sim.set_words(host[:n0], step0)      # H2D of the inputs (pinned)
            for _ in range(k):
                sim.step(1)
                sim.stats()                      # D2H of the step's metric (counters)
            n1 = sim.read_state(words=host)      # D2H of the result
            t1 = time.perf_counter()
            e2e_s = t1 - t0
            nt = n0
            if world > 1:
                t = torch.tensor([e2e_s], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                e2e_s = float(t.item())
                c = torch.tensor([n0], device="cuda", dtype=torch.int64)
                dist.all_reduce(c)
                nt = int(c.item())
            stats_bytes = 8 * (2 + 3 * 64 + 5)
            e2e = {"value": nt * k / e2e_s, "unit": "particle-steps/s",
                   "h2d_bytes_per_step": int(n0 * W * 4 / k),
                   "d2h_bytes_per_step": int(n1 * W * 4 / k + stats_bytes),
                   "note": f"timed: set_words(pinned host, {n0*W*4/1e9:.2f} GB) + {k} x (qmpm_step + qmpm_stats D2H) "
                           "+ read_state(words -> pinned host); rank 0's bytes"}
            del host
        sim.close()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---------------- roofline of the dominant kernel
    import json as _json
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peaks = _json.load(open(peaks_path))
        hbm_peak, peak_src = float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        hbm_peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    S = W * 4
    nodes = 64 * int(st.touched_blocks)
    ab = algorithmic_bytes(S, nodes)
    dom = max(("p2g", "g2p", "grid_update"), key=lambda k: ktimes[k][0])
    kms, kcnt = ktimes[dom]
    avg_ms = kms / max(kcnt, 1)
    achieved = ab[dom](N) / (avg_ms / 1e3) / 1e9
    # ncu `--set full` capture of this config's kernels (profiles/ncu_traffic.json, written
    # by profiles/summarize_ncu.py --config): DRAM bytes and warp instructions per launch
    traffic, winst, fma_frac = None, None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath) and not args.n and args.scaling == "weak" and args.z_extent == 1.0:
        try:
            rec = _json.load(open(tpath)).get(args.config, {}).get(dom, {})
            traffic, winst, fma_frac = rec.get("traffic"), rec.get("warp_inst"), rec.get("fma_pipe")
        except Exception:
            traffic, winst, fma_frac = None, None, None
    # issue-rate roofline: the step kernels are bound by the warp
    # schedulers, not by bytes -- warp instructions per launch / (launch time x SMs x 4
    # schedulers x SM clock under load)
    issue_frac = None
    if winst and clk and clk.get("sm_mhz"):
        n_sm = torch.cuda.get_device_properties(local).multi_processor_count
        issue_frac = winst / (avg_ms * 1e-3 * n_sm * 4 * clk["sm_mhz"] * 1e6)
    step_ms = ms / args.steps
    B_alg = 2 * S + 56.0 * nodes / N  # SURVEY §8(d) M3 per particle-step
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": ab[dom](N), "avg_launch_ms": avg_ms,
                "issue_frac": issue_frac,
                "issue_note": "warp instructions per launch (ncu, profiles/ncu_traffic.json, this config) / "
                              "(avg launch time x SMs x 4 schedulers x median SM clock): the binding roofline "
                              "of the issue-bound step kernels (SURVEY §8(d) M4)",
                "fma_pipe_frac": fma_frac,
                "fma_pipe_note": "ncu sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active of this kernel "
                                 "(this config): FFMA/FMUL/FADD, their packed FP32x2 forms and IMAD share the FMA "
                                 "pipe at one warp instruction per 2 cycles per scheduler -- the unit that binds "
                                 "P2G and G2P (DESIGN.md §6)"}
    kshare = {k: {"ms_per_step": v[0] / max(v[1], 1) * (v[1] / args.steps), "launches": v[1]}
              for k, v in ktimes.items()}

    # ---------------- CPU oracle baseline (rank 0, N = 1)
    cpu = None
    if world == 1:
        rate1, n_s, s_s, secs1, _ = cpu_oracle_rate(sc, sch, args.cpu_sample, args.cpu_steps, threads=1)
        rate, n_m, s_m, secs, used = cpu_oracle_rate(sc, sch, args.cpu_sample, 4 * args.cpu_steps, threads=0)
        cpu = {"value": rate, "unit": "particle-steps/s", "cores": used, "kind": "oracle",
               "sample": f"first {n_m:,} particles of the workload, {s_m} steps from the initial state "
                         f"(fp64 plain C, OpenMP particle loops on {used} threads, {secs:.1f} s)",
               "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
               "single_thread": {"value": rate1, "cores": 1,
                                 "sample": f"first {n_s:,} particles, {s_s} steps ({secs1:.1f} s)"}}

    line = {
        "metric": "quantized MPM particle-steps/sec", "value": value, "unit": "particle-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": (value / (world if args.scaling == "weak" else 1) / PAPER_PSTEPS[args.config])
        if (args.config in PAPER_PSTEPS and not args.n and args.layout == "pack"
            and scheme_name(args) == {"c3": "e0.01", "c4": "f2"}[args.config])
        else None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(args, sc, W, bits), "particles_per_gpu": N,
                   "particles_total": sc.n_particles,
                   "scheme": scheme_name(args), "record_bytes": S, "rounding": args.rounding,
                   "round_counters": not args.no_counters, "scene_warmup_steps": args.scene_warmup,
                   "l2": (f"state {N * S / 1e9:.1f} GB per buffer >> 126 MB L2: no flush needed"
                          if N * S > 1e9 else
                          f"state {N * S / 1e6:.1f} MB fits in L2 and is not flushed: a launch/latency-bound "
                          "side line (BASELINE configs[0]/[1]), not the headline"),
                   "parallelism": "single GPU" if world == 1 else
                   f"z-slab decomposition over {world} GPUs (ghost-plane + velocity halo + migration over NCCL)",
                   "baseline_ref": "vs_baseline = per-GPU value / the paper's RTX 3090 T-large rate for this workload "
                                   "(derived: C3 5.95e8, C4 3.68e8 p-steps/s, P:945-946): context, not a target"},
        "roofline": roofline,
        "hbm_roofline_step": {"bytes_per_particle_step": B_alg,
                              "achieved_GBps": value / world * B_alg / 1e9,
                              "frac_of_8TBps": value / world * B_alg / 8e12,
                              "frac_of_measured": value / world * B_alg / (hbm_peak * 1e9)},
        "kernels": kshare,
        "active_blocks": int(st.active_blocks), "touched_blocks": int(st.touched_blocks),
        "out_of_domain": int(st.out_of_domain), "nonfinite": int(st.nonfinite), "pool_overflow": int(st.pool_overflow),
        "gpu_launches": int(launches),
        "e2e": e2e,
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.scene_warmup is None:
        args.scene_warmup = DEFAULT_SCENE_WARMUP[args.config]
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
