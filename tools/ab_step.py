"""Paired A/B of step-kernel variants on ONE developed state (tuning only, GPU box).

The C4 scene is advanced `--warm` steps once; its packed words are kept on the device and
every variant (NVRTC options in QMPM_JIT_OPTS, e.g. -DQMPM_AB_ZPACK=0) starts from them:
kernel times over --steps steps with per-launch events, the baseline repeated first and
last.  Prints one line per variant.

    python tools/ab_step.py --warm 2000 --steps 20 --variant=-DQMPM_AB_ZPACK=0 --variant=ENV:QMPM_G2P_MINB=3 ...
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_04658_b200 import qmpm, scenes, schemes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--warm", type=int, default=2000)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--config", default="c4")
ap.add_argument("--no-counters", action="store_true")
ap.add_argument("--variant", action="append", default=[], help="NVRTC options of one variant (use --variant=...)")
a = ap.parse_args()
if a.config == "c3":
    sc, sch = scenes.c3(), schemes.e001()
elif a.config == "c4_8ppc":
    sc, sch = scenes.c4(res=512, dt=5e-5), schemes.f2()
else:
    sc, sch = scenes.c4(), schemes.f2()
flags = qmpm.NO_ROUND_COUNTERS if a.no_counters else 0
stream = torch.cuda.Stream()
N = sc.n_particles
with torch.cuda.stream(stream):
    os.environ.pop("QMPM_JIT_OPTS", None)
    sim = qmpm.Sim(sc.sim, sch, N, flags=flags, stream=stream)
    for s0 in range(0, N, 1 << 24):
        st = sc.state_chunk(s0, min(1 << 24, N - s0), backend="torch", device="cuda")
        (sim.set_state if s0 == 0 else sim.append_state)(st)
        stream.synchronize()
    sim.step(a.warm)
    words = torch.empty((N, sim.W), dtype=torch.int32, device="cuda")
    sim.read_state(words=words)
    step0 = sim.stats().step
    sim.close()
    del sim
    torch.cuda.empty_cache()

    def measure(opts):
        # "ENV:NAME=VALUE[,NAME=VALUE]" sets environment variables (e.g. QMPM_G2P_MINB) instead
        envs = {}
        if opts.startswith("ENV:"):
            envs = dict(kv.split("=", 1) for kv in opts[4:].split(","))
            opts = ""
        for k in ("QMPM_G2P_MINB", "QMPM_P2G_MINB"):
            os.environ.pop(k, None)
        os.environ.update(envs)
        if opts:
            os.environ["QMPM_JIT_OPTS"] = opts
        else:
            os.environ.pop("QMPM_JIT_OPTS", None)
        s = qmpm.Sim(sc.sim, sch, N, flags=flags, stream=stream)
        s.set_words(words, step0)
        s.step(3)
        s.set_profiling(True)
        s.step(a.steps)
        kt = s.kernel_times()
        s.close()
        return {k: v[0] / max(v[1], 1) for k, v in kt.items() if v[1]}

    for v in [""] + a.variant + [""]:
        k = measure(v)
        tot = sum(k.values())
        print(f"{v or 'baseline':45s} step {tot:7.3f} ms  g2p {k.get('g2p', 0):7.3f}  p2g {k.get('p2g', 0):7.3f}  "
              f"scatter {k.get('bin_scatter', 0):6.3f}", flush=True)
