"""GPU tests of the slab decomposition with the in-process
transport (qmpm_step_group): k z-slabs on one GPU exchange ghost planes, velocity
planes and migrating particles exactly as the NCCL transport does between GPUs.

The slab run must meet the SAME parity bar as the single-GPU run: one step from
oracle-generated words vs the fp64 oracle within 1e-5 on the conditioning-aware
scales, and the stored words bit-exact to the oracle codec on the GPU's own floats
(content-keyed dithering makes codes independent of the rank that stores them)."""
import numpy as np
import pytest

import oracle
from paper_2207_04658_b200 import qmpm, scenes, schemes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from test_gpu_step import REL, scales  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def cuts(nz, k):
    """k slabs of whole 4-cell block planes"""
    nb = nz // 4
    b = [round(i * nb / k) * 4 for i in range(k + 1)]
    b[-1] = nz
    return list(zip(b[:-1], b[1:]))


def owner(state, sim, slabs):
    z = np.floor(state[:, 2].astype(np.float64) / sim["dx"] - 0.5).astype(np.int64)
    z = np.clip(z, 0, sim["grid_res"][2] - 3)
    o = np.zeros(len(z), np.int64)
    for r, (z0, z1) in enumerate(slabs):
        o[(z >= z0) & (z < z1)] = r
    return o


def make_group(sc, sch, words, step0, k, flags, mig_caps=None):
    slabs = cuts(sc.sim["grid_res"][2], k)
    st = oracle.decode_state(sch, words)
    own = owner(st, sc.sim, slabs)
    stream = torch.cuda.Stream()
    sims = []
    for r, (z0, z1) in enumerate(slabs):
        idx = np.nonzero(own == r)[0]
        s = qmpm.Sim(sc.sim, sch, words.shape[0], flags=flags, stream=stream, slab=(k, r, z0, z1),
                     migrate_capacity=mig_caps[r] if mig_caps else 0)
        s.set_words(dev(words[idx]), step0)
        s.set_ids(dev(idx.astype(np.uint32)))
        sims.append(s)
    return sims, slabs


def gather(sims, ns, W, debug=True):
    pre, words, ids = [], [], []
    for s in sims:
        n = s.stats().n_particles
        w = np.zeros((n, W), np.uint32)
        i = np.zeros(n, np.uint32)
        s.read_state(words=w, ids=i, capacity=n)
        words.append(w)
        ids.append(i)
        if debug:
            p = np.zeros((n, ns), np.float32)
            s.read_debug(p)
            pre.append(p)
    ids = np.concatenate(ids)
    order = np.argsort(ids)
    out_pre = np.concatenate(pre)[order] if debug else None
    return ids[order], np.concatenate(words)[order], out_pre


@pytest.mark.parametrize("k", [2, 3])
@pytest.mark.parametrize("case", ["fluid", "elastic", "fluid_res32"])
def test_slab_step_matches_oracle(case, k):
    if case == "fluid":
        sc, sch = scenes.small_fluid_3d(), schemes.f2()
    elif case == "fluid_res32":  # slab block tables of one scan tile: the fused sort front
        sc, sch = scenes.small_fluid_3d(res=32, n_target=20_000), schemes.f2()
    else:
        sc, sch = scenes.small_elastic_3d(), schemes.e01()
    w0, _ = oracle.encode_state(sch, sc.state())
    w_in, _ = oracle.run(sc.sim, sch, w0, 1, 10)
    o_pre, o_words, _ = oracle.step(sc.sim, sch, w_in, 11)
    sims, slabs = make_group(sc, sch, w_in, 10, k, qmpm.TRACK_IDS | qmpm.DEBUG_PREENCODE)
    qmpm.step_group(sims, 1)
    ids, g_words, g_pre = gather(sims, sims[0].n_scalars, sims[0].W)
    for s in sims:
        s.close()
    n = w_in.shape[0]
    assert np.array_equal(ids, np.arange(n))  # every particle exactly once
    s_h = scales(sc.sim, o_pre, oracle.decode_state(sch, w_in))
    err = np.abs(g_pre.astype(np.float64) - o_pre) / np.maximum(np.abs(o_pre), s_h)
    assert err.max() <= REL, err.max(axis=0)
    keys = np.array([oracle.particle_key(sch, w_in[i]) for i in range(n)], np.uint32)
    assert np.array_equal(g_words, oracle.encode_state(sch, g_pre, step=11, keys=keys)[0])


def test_ranks_agree_on_one_migration_capacity():
    """The migration exchanges are fixed-size, so ranks whose capacities differ (the
    default follows each rank's particle capacity, which differs between slabs) are
    re-sized to the largest before the first exchange -- the in-process group here, the
    NCCL connect by an all-reduce -- instead of posting mismatched transfers."""
    sc, sch = scenes.small_fluid_3d(), schemes.f2()
    w0, _ = oracle.encode_state(sch, sc.state())
    w_in, _ = oracle.run(sc.sim, sch, w0, 1, 10)
    o_pre, _, _ = oracle.step(sc.sim, sch, w_in, 11)
    sims, _ = make_group(sc, sch, w_in, 10, 3, qmpm.TRACK_IDS | qmpm.DEBUG_PREENCODE,
                         mig_caps=[65536, 90000, 70000])
    qmpm.step_group(sims, 1)
    ids, _, g_pre = gather(sims, sims[0].n_scalars, sims[0].W)
    for s in sims:
        s.close()
    assert np.array_equal(ids, np.arange(w_in.shape[0]))
    s_h = scales(sc.sim, o_pre, oracle.decode_state(sch, w_in))
    err = np.abs(g_pre.astype(np.float64) - o_pre) / np.maximum(np.abs(o_pre), s_h)
    assert err.max() <= REL, err.max(axis=0)


def test_slab_run_conserves_and_matches_single_gpu():
    """20 steps of a 3-slab group vs one context: particle count conserved, every
    particle stored by the rank owning its slab, KE/COM within 1e-3 (P3)."""
    sc, sch = scenes.small_fluid_3d(), schemes.f2()
    st0 = sc.state()
    w0, _ = oracle.encode_state(sch, st0)
    sims, slabs = make_group(sc, sch, w0, 0, 3, qmpm.TRACK_IDS)
    qmpm.step_group(sims, 20)
    ids, g_words, _ = gather(sims, sims[0].n_scalars, sims[0].W, debug=False)
    for r, s in enumerate(sims):
        n = s.stats().n_particles
        w = np.zeros((n, s.W), np.uint32)
        s.read_state(words=w, capacity=n)
        st = oracle.decode_state(sch, w)
        assert np.all(owner(st, sc.sim, slabs) == r)
        s.close()
    assert np.array_equal(ids, np.arange(st0.shape[0]))
    one = qmpm.Sim(sc.sim, sch, st0.shape[0])
    one.set_words(dev(w0), 0)
    one.step(20)
    w1 = np.zeros_like(w0)
    one.read_state(words=w1)
    one.close()
    ke_g, com_g = oracle.aggregates(sc.sim, oracle.decode_state(sch, g_words))
    ke_1, com_1 = oracle.aggregates(sc.sim, oracle.decode_state(sch, w1))
    assert abs(ke_g - ke_1) <= 1e-3 * abs(ke_1)
    assert np.all(np.abs(com_g - com_1) <= 1e-3 * np.abs(com_1))


def test_slab_validation():
    sc, sch = scenes.small_fluid_3d(), schemes.f2()
    with pytest.raises(qmpm.QmpmError):
        qmpm.Sim(sc.sim, sch, 10, slab=(2, 0, 0, 30))  # not on a block plane
    with pytest.raises(qmpm.QmpmError):
        qmpm.Sim(sc.sim, sch, 10, slab=(2, 2, 0, 32))  # bad rank
    s = qmpm.Sim(sc.sim, sch, 10, slab=(2, 0, 0, 32))
    with pytest.raises(qmpm.QmpmError) as e:
        s.step(1)  # no transport
    assert e.value.code == 9
    s.close()


def test_migration_overflow_is_a_sticky_error_not_a_hang():
    """A migration buffer too small for the step's leavers (migrate_capacity = 1): the
    exchange still runs its fixed schedule (no rank waits on a count), the device status
    becomes ECAPACITY at the next synchronising call, and further steps are refused until
    the state is set again (SURVEY §8(b) error semantics)."""
    sc, sch = scenes.small_fluid_3d(), schemes.f2()
    w0, _ = oracle.encode_state(sch, sc.state())
    slabs = cuts(sc.sim["grid_res"][2], 2)
    st = oracle.decode_state(sch, w0)
    own = owner(st, sc.sim, slabs)
    stream = torch.cuda.Stream()
    sims = []
    for r, (z0, z1) in enumerate(slabs):
        idx = np.nonzero(own == r)[0]
        s = qmpm.Sim(sc.sim, sch, w0.shape[0], stream=stream, slab=(2, r, z0, z1), migrate_capacity=1)
        # everything to rank 0: rank 1's particles must all migrate (far more than 1)
        s.set_words(dev(w0[idx]), 0)
        sims.append(s)
    # rank 1 gets particles of rank 0's top block plane (one hop down): its first step
    # routes thousands of them into a buffer of one record
    zb = np.floor(st[:, 2].astype(np.float64) / sc.sim["dx"] - 0.5).astype(np.int64)
    top0 = np.nonzero((own == 0) & (zb >= slabs[0][1] - 4))[0]
    assert top0.size > 100
    sims[1].set_words(dev(w0[top0]), 0)
    qmpm.step_group(sims, 1)  # returns: fixed schedule, no hang
    with pytest.raises(qmpm.QmpmError) as e:
        sims[1].stats()
    assert e.value.code == 8  # ECAPACITY
    with pytest.raises(qmpm.QmpmError) as e:
        qmpm.step_group(sims, 1)
    assert e.value.code == 9  # ESTATE until set_state / set_words
    for s in sims:
        s.close()


def test_nonfinite_state_is_reported():
    """a non-finite value is an error value -- it is encoded as code 0 and counted,
    and read_state reports QMPM_ENONFINITE (the state is still read)."""
    sc, sch = scenes.small_fluid_3d(), schemes.f2()
    st = sc.state()
    st[7, 3] = np.nan
    sim = qmpm.Sim(sc.sim, sch, st.shape[0])
    sim.set_state(dev(st))
    w = np.zeros((st.shape[0], sim.W), np.uint32)
    with pytest.raises(qmpm.QmpmError) as e:
        sim.read_state(words=w)
    assert e.value.code == 6
    assert oracle.decode_state(sch, w[7:8])[0, 3] == 0.0
    sim.set_state(dev(sc.state()))  # a fresh state clears it
    sim.read_state(words=w)
    sim.close()


def test_two_slab_jump_is_edomain():
    """A particle handed to a rank two slabs away from its owner cannot be routed in one
    hop (CFL keeps migration to the neighbours): the next synchronising call reports
    QMPM_EDOMAIN (sticky), never a hang."""
    sc, sch = scenes.small_fluid_3d(), schemes.f2()
    w0, _ = oracle.encode_state(sch, sc.state())
    slabs = cuts(sc.sim["grid_res"][2], 3)
    st = oracle.decode_state(sch, w0)
    own = owner(st, sc.sim, slabs)
    stream = torch.cuda.Stream()
    sims = []
    for r, (z0, z1) in enumerate(slabs):
        idx = np.nonzero(own == r)[0]
        s = qmpm.Sim(sc.sim, sch, w0.shape[0], stream=stream, slab=(3, r, z0, z1))
        s.set_words(dev(w0[idx]), 0)
        sims.append(s)
    sims[2].set_words(dev(w0[np.nonzero(own == 0)[0][:100]]), 0)  # rank 0's particles on rank 2
    qmpm.step_group(sims, 1)
    with pytest.raises(qmpm.QmpmError) as e:
        sims[2].stats()
    assert e.value.code == 7  # EDOMAIN
    for s in sims:
        s.close()
