"""Algorithm 1 end to end on the GPU (the paper's error-bounded experiment, P:563-630,
on the C1 scene): an fp32 run records the ranges (Alg. 1 line 9), the gradient tallies
g_h come from the adjoint with bisection checkpointing (line 12), the closed form gives
(b_h, R_h) for an error bound eps (lines 13-15), and the quantized run's final kinetic
energy is compared with the fp32 run's: success when |z_q - z| <= eps z.

    python tools/alg1_error_bounded.py [--steps 2048] [--eps 0.1 0.05 0.01] [--seeds 3] [--mem 0.5 0.4 0.3]

Also the memory-bounded scheme (Eq. 7) for budgets of --mem x the fp32 state.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(T, eps_list, seeds, mem_ratios=()):
    import numpy as np
    import torch
    from paper_2207_04658_b200 import qadjoint, qmpm, scenes, schemes

    sc = scenes.c1()
    st = sc.state()
    n = st.shape[0]
    d = sc.sim["dim"]
    m = sc.sim["p_rho"] * sc.sim["p_vol"]

    def ke(s):
        return 0.5 * m * float(np.sum(s[:, d:2 * d].astype(np.float64) ** 2))

    # fp32 run with range recording
    sim = qmpm.Sim(sc.sim, schemes.fp32(d), n, flags=qmpm.RECORD_RANGES)
    sim.set_state(torch.from_numpy(st).cuda())
    sim.step(T)
    max_abs = sim.read_ranges()
    s32 = np.zeros(st.shape, np.float32)
    sim.read_state(vals=s32)
    sim.close()
    z = ke(s32)
    # gradient tallies (the same fp32 physics on the adjoint engine's dense grid)
    A = qadjoint.Adjoint(sc.sim, n)
    g, z_adj, stats = A.gradient_tally(torch.from_numpy(st).cuda(), T)
    A.close()
    R = schemes.ranges_from_record(max_abs)
    P = np.full(len(R), float(n))
    rows = []
    for eps in eps_list:
        delta, bits = qmpm.solve_error_bounded(P, np.maximum(g, 1e-300), R, z, eps, b_min=1, b_max=31)
        sigma = qmpm.predict_error(delta, g)
        sch = schemes.from_solution(d, "elastic", R, bits)
        _, W, nbits = qmpm.layout(sch)
        for seed in range(seeds):
            sch_s = dict(sch, seed=schemes.DITHER_SEED + seed)
            q = qmpm.Sim(sc.sim, sch_s, n)
            q.set_state(torch.from_numpy(st).cuda())
            q.step(T)
            sq = np.zeros(st.shape, np.float32)
            q.read_state(vals=sq)
            stq = q.stats()
            q.close()
            zq = ke(sq)
            rows.append(dict(eps=eps, seed=seed, z_fp32=z, z_quant=zq, rel_err=abs(zq - z) / z,
                             success=abs(zq - z) <= eps * z, sigma_pred=sigma, bits=[int(b) for b in bits],
                             record_bits=nbits, compression=32.0 * len(bits) / nbits,
                             saturations=int(sum(stq.saturations))))
    # the same schemes rounded to nearest instead of dithered (the paper's dithering
    # comparison: without dithering the errors correlate and bias z)
    rne_rows = []
    for eps in eps_list:
        delta, bits = qmpm.solve_error_bounded(P, np.maximum(g, 1e-300), R, z, eps, b_min=1, b_max=31)
        sch = schemes.with_rounding(schemes.from_solution(d, "elastic", R, bits), "rne")
        q = qmpm.Sim(sc.sim, sch, n)
        q.set_state(torch.from_numpy(st).cuda())
        q.step(T)
        sq = np.zeros(st.shape, np.float32)
        q.read_state(vals=sq)
        q.close()
        zq = ke(sq)
        rne_rows.append(dict(eps=eps, z_quant=zq, rel_err=abs(zq - z) / z, success=abs(zq - z) <= eps * z))
    # memory-bounded (Eq. 7): stored bits <= ratio x fp32 (32 bits per scalar)
    mem_rows = []
    for ratio in mem_ratios:
        H = len(R)
        budget = ratio * 32.0 * H * n - float(H * n)  # fraction bits (stored width = bits + 1)
        delta, bits = qmpm.solve_memory_bounded(P, np.maximum(g, 1e-300), R, budget, b_min=1, b_max=31)
        sigma = qmpm.predict_error(delta, g)
        sch = schemes.from_solution(d, "elastic", R, bits)
        _, W, nbits = qmpm.layout(sch)
        for seed in range(seeds):
            q = qmpm.Sim(sc.sim, dict(sch, seed=schemes.DITHER_SEED + seed), n)
            q.set_state(torch.from_numpy(st).cuda())
            q.step(T)
            sq = np.zeros(st.shape, np.float32)
            q.read_state(vals=sq)
            stq = q.stats()
            q.close()
            zq = ke(sq)
            mem_rows.append(dict(ratio=ratio, seed=seed, z_quant=zq, rel_err=abs(zq - z) / z,
                                 sigma_pred_rel=sigma / z, bits=[int(b) for b in bits], record_bits=nbits,
                                 compression=32.0 * len(bits) / nbits, saturations=int(sum(stq.saturations))))
    return dict(scene="C1 (2D elastic, 8192 particles, 128^2, dt 2e-4)", steps=T, z_fp32=z, z_adjoint_engine=z_adj,
                g=[float(x) for x in g], ranges=[float(r) for r in R], checkpointing=stats, runs=rows,
                rne=rne_rows, memory_bounded=mem_rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2048)
    ap.add_argument("--eps", type=float, nargs="+", default=[0.1, 0.05, 0.01])
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--mem", type=float, nargs="*", default=[0.5, 0.4, 0.3], help="memory-bounded ratios of fp32")
    a = ap.parse_args()
    print(json.dumps(run(a.steps, a.eps, a.seeds, a.mem)), flush=True)


if __name__ == "__main__":
    main()
