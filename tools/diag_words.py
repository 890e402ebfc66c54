"""Diagnose a G2P word mismatch: one GPU step from oracle-warmed words; compare the
stored codes with the oracle codec applied to the GPU's pre-encode floats."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2207_04658_b200 import qmpm, scenes, schemes  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "f2"
sc = scenes.small_fluid_3d() if case == "f2" else scenes.small_elastic_3d()
sch = schemes.f2() if case == "f2" else schemes.e001()
w0, _ = oracle.encode_state(sch, sc.state())
w_in, _ = oracle.run(sc.sim, sch, w0, 1, 20)
n = w_in.shape[0]
sim = qmpm.Sim(sc.sim, sch, n, flags=qmpm.TRACK_IDS | qmpm.DEBUG_PREENCODE)
sim.set_words(torch.from_numpy(w_in.view(np.int32)).cuda(), 20)
sim.step(1)
pre = np.zeros((n, sim.n_scalars), np.float32)
words = np.zeros_like(w_in)
ids = np.zeros(n, np.uint32)
sim.read_state(words=words, ids=ids)
sim.read_debug(pre)
sim.close()
inv = np.argsort(ids)
pre, words = pre[inv], words[inv]
keys = np.array([oracle.particle_key(sch, w_in[i]) for i in range(n)], np.uint32)
ref, _ = oracle.encode_state(sch, pre, step=21, keys=keys)
dg = oracle.decode_state(sch, words)
dr = oracle.decode_state(sch, ref)
bad = dg != dr
print("records differing:", int(bad.any(axis=1).sum()), "of", n, "; per scalar:", bad.sum(axis=0).tolist())
rows = np.nonzero(bad.any(axis=1))[0][:8]
for r in rows:
    c = np.nonzero(bad[r])[0]
    print(r, [(int(i), float(pre[r, i]), float(dg[r, i]), float(dr[r, i])) for i in c])
