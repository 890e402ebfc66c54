"""How often are a G2P chunk's 32 records contiguous in memory (the precondition of one
bulk/TMA copy per chunk instead of per-lane copies)?  Records are stored in the previous
step's (block, cell) order; the next step's chunk takes 32 consecutive particles of the
new order.  Measured on oracle-advanced states at C4 and C3 densities (host only).

    python tools/record_contiguity.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2207_04658_b200 import scenes, schemes  # noqa: E402


def keys(sim, st):
    base = np.floor(st[:, :3].astype(np.float64) / sim["dx"] - 0.5).astype(np.int64)
    b, c = base >> 2, base & 3
    return ((b[:, 2] * 4096 + b[:, 0]) * 4096 + b[:, 1]) * 64 + (c[:, 0] * 16 + c[:, 1] * 4 + c[:, 2])


for name, sc, sch in (("C4 density (fluid, ~55 ppc)", scenes.developed_fluid(), schemes.f2()),
                      ("C3 density (elastic, 8 ppc)", scenes.colliding_elastic(cube=18), schemes.e001())):
    w, _ = oracle.encode_state(sch, sc.state())
    w, _ = oracle.run(sc.sim, sch, w, 1, 60, threads=0)
    s0 = oracle.decode_state(sch, w)
    order0 = np.argsort(keys(sc.sim, s0), kind="stable")       # storage order after step t
    w1, _ = oracle.run(sc.sim, sch, w[order0], 61, 1, threads=0)
    s1 = oracle.decode_state(sch, w1)
    k1 = keys(sc.sim, s1)
    perm = np.argsort(k1, kind="stable")                         # slot of the j-th particle of the new order
    blk = k1[perm] >> 6
    starts = np.concatenate([[0], np.nonzero(np.diff(blk))[0] + 1, [len(blk)]])
    tot = cont = 0
    for a, b in zip(starts[:-1], starts[1:]):
        for j0 in range(a, b, 32):
            p = perm[j0:min(j0 + 32, b)]
            tot += 1
            cont += bool(np.all(np.diff(p) == 1))
    print(f"{name}: {cont}/{tot} chunks contiguous ({100.0 * cont / tot:.1f} %)")
