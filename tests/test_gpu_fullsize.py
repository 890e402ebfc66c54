"""P2 parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(C4: 400M fluid particles on 256^3, F2; C3: 295M elastic particles on 1024^3, E0.01):
one step from the seeded initial state on the GPU, then a sample of particles is
checked against the oracle one by one.  The oracle's input for a sampled particle is
its lattice neighbourhood (every particle within 3.5 cells, generated and encoded on
the host by the same seeded scene generator -- never read from the GPU), which holds
every particle that reaches the sampled particle's stencil nodes, so its sampled step
(oracle_step_sampled_f64) is exact for that particle."""
import math

import numpy as np
import pytest

import oracle
from paper_2207_04658_b200 import qmpm, scenes, schemes
from test_gpu_step import REL, scales

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")


def neighbourhood(sc, gid, cells=3.5):
    """Global indices of the lattice neighbourhood (+-cells grid cells) of particle gid,
    and the position of gid in that list."""
    first = 0
    for b in sc.boxes:
        nb = b.size()
        if gid < first + nb:
            break
        first += nb
    nx, ny, nz = b.counts
    loc = gid - first
    i, j, k = loc // (ny * nz), (loc // nz) % ny, loc % nz
    m = int(math.ceil(cells * sc.sim["dx"] / b.spacing)) + 1
    out = []
    for ii in range(max(0, i - m), min(nx, i + m + 1)):
        for jj in range(max(0, j - m), min(ny, j + m + 1)):
            lo = (ii * ny + jj) * nz + max(0, k - m)
            hi = min((ii * ny + jj) * nz + min(nz, k + m + 1), nb)
            if lo < hi:
                out.append(np.arange(first + lo, first + hi, dtype=np.int64))
    idx = np.concatenate(out)
    return idx, int(np.nonzero(idx == gid)[0][0])


def host_state(sc, idx):
    runs = np.split(idx, np.nonzero(np.diff(idx) != 1)[0] + 1)
    return np.concatenate([sc.state_chunk(int(r[0]), len(r)) for r in runs])


@pytest.mark.parametrize("config", ["c4", "c3"])
def test_full_size_sampled_step(config):
    if config == "c4":
        sc, sch = scenes.c4(), schemes.f2()
    else:
        sc, sch = scenes.c3(), schemes.e001()
    N = sc.n_particles
    ns = sc.n_scalars
    sim = qmpm.Sim(sc.sim, sch, N, flags=qmpm.TRACK_IDS | qmpm.DEBUG_PREENCODE)
    chunk = 1 << 24
    for s0 in range(0, N, chunk):
        st = sc.state_chunk(s0, min(chunk, N - s0), backend="torch", device="cuda")
        (sim.set_state if s0 == 0 else sim.append_state)(st)
        torch.cuda.synchronize()
        del st
    sim.step(1)
    assert sim.stats().n_particles == N
    rng = np.random.default_rng(7)
    sample = np.sort(rng.choice(N, 16, replace=False))
    ids = torch.empty(N, dtype=torch.int32, device="cuda")
    words = torch.empty((N, sim.W), dtype=torch.int32, device="cuda")
    sim.read_state(words=words, ids=ids)
    inv = torch.empty(N, dtype=torch.int64, device="cuda")
    inv[ids.long()] = torch.arange(N, dtype=torch.int64, device="cuda")
    rows = inv[torch.from_numpy(sample).cuda()]
    del inv, ids
    g_words = words[rows].cpu().numpy().view(np.uint32)
    del words
    pre = torch.empty((N, ns), dtype=torch.float32, device="cuda")
    sim.read_debug(pre)
    g_pre = pre[rows].cpu().numpy()
    del pre
    sim.close()
    torch.cuda.empty_cache()

    for q, gid in enumerate(sample):
        idx, me = neighbourhood(sc, int(gid))
        st = host_state(sc, idx)
        w0, _ = oracle.encode_state(sch, st)  # qmpm_set_state: RNE at step 0 (reading Q20)
        o_pre, _ = oracle.step_sampled(sc.sim, sch, w0, 1, np.array([me], np.uint64))
        s = scales(sc.sim, o_pre, oracle.decode_state(sch, w0))
        err = np.abs(g_pre[q].astype(np.float64) - o_pre[0]) / np.maximum(np.abs(o_pre[0]), s)
        assert err.max() <= REL, (config, int(gid), err)
        key = np.array([oracle.particle_key(sch, w0[me])], np.uint32)
        w_ref, _ = oracle.encode_state(sch, g_pre[q:q + 1], step=1, keys=key)
        assert np.array_equal(g_words[q], w_ref[0]), (config, int(gid))
