"""GPU: range recording (Algorithm 1 line 9) and the scheme-derivation pipeline
of SURVEY §8(f) row f2 (record ranges on the full-precision run, solve, run quantized)."""
import numpy as np
import pytest

import oracle
from oracle import solver as osol
from paper_2207_04658_b200 import qmpm, scenes, schemes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("case", ["c1", "fluid"])
def test_record_ranges_equal_max_of_preencode_state(case):
    sc = scenes.c1() if case == "c1" else scenes.small_fluid_3d()
    sch = schemes.x16() if case == "c1" else schemes.f2()
    st = sc.state()
    n = st.shape[0]
    sim = qmpm.Sim(sc.sim, sch, n, flags=qmpm.RECORD_RANGES | qmpm.DEBUG_PREENCODE)
    sim.set_state(dev(st))
    pre = np.zeros((n, sim.n_scalars), np.float32)
    run_max = np.zeros(sim.n_scalars, np.float32)
    for t in range(4):
        sim.step(1)
        sim.read_debug(pre)
        step_max = np.abs(pre).max(axis=0)
        run_max = np.maximum(run_max, step_max)
        r = sim.read_ranges(reset=(t == 2))
        np.testing.assert_array_equal(r, step_max if t == 3 else run_max)
        if t == 2:
            run_max[:] = 0.0
    sim.close()


@pytest.mark.parametrize("case", ["c1", "fluid", "elastic"])
def test_record_ranges_match_oracle_preencode_maxima(case):
    """Alg. 1 line 9 against the ORACLE: one step from oracle-warmed words; the recorded
    max |value| per state scalar equals the maximum over particles of the fp64 oracle's
    pre-encode state within the P2 tolerance of the values (1e-5 of the conditioning-aware
    scale): a range recorded from the wrong stage (decoded input, post-encode) or the
    wrong scalar misses it by far more."""
    from test_gpu_step import REL, scales
    if case == "c1":
        sc, sch = scenes.c1(), schemes.x16()
    elif case == "fluid":
        sc, sch = scenes.small_fluid_3d(), schemes.f2()
    else:
        sc, sch = scenes.small_elastic_3d(), schemes.e01()
    w0, _ = oracle.encode_state(sch, sc.state())
    w_in, _ = oracle.run(sc.sim, sch, w0, 1, 12)
    o_pre, _, _ = oracle.step(sc.sim, sch, w_in, 13)
    n = w_in.shape[0]
    sim = qmpm.Sim(sc.sim, sch, n, flags=qmpm.RECORD_RANGES)
    sim.set_words(dev(w_in.view(np.int32)), 12)
    sim.step(1)
    r = sim.read_ranges(reset=True).astype(np.float64)
    sim.close()
    o_max = np.abs(o_pre).max(axis=0)
    s_h = scales(sc.sim, o_pre, oracle.decode_state(sch, w_in))
    assert np.all(np.abs(r - o_max) <= REL * np.maximum(o_max, s_h)), (r, o_max)
    # and it is not the decoded input's maximum (the state did change)
    i_max = np.abs(oracle.decode_state(sch, w_in)).max(axis=0)
    assert np.any(np.abs(i_max - o_max) > REL * np.maximum(o_max, s_h))


def test_scheme_derivation_pipeline():
    """Algorithm 1 without the adjoint (g_h supplied): ranges recorded by the fp32 run
    (x2, power of two), fraction bits from the error-bounded closed form, then the
    quantized run of the same scene: it stores without saturating, its kinetic energy
    stays within the fp32 run's by 2 %, and the library's bits equal the oracle's."""
    sc = scenes.c1()
    st = sc.state()
    n = st.shape[0]
    steps = 60
    f32 = schemes.fp32(2)
    sim = qmpm.Sim(sc.sim, f32, n, flags=qmpm.RECORD_RANGES)
    sim.set_state(dev(st))
    sim.step(steps)
    max_abs = sim.read_ranges()
    s32 = np.zeros(st.shape, np.float32)
    sim.read_state(vals=s32)
    sim.close()
    ke32, _ = oracle.aggregates(sc.sim, s32)
    R = schemes.ranges_from_record(max_abs)
    H = len(R)
    P = np.full(H, float(n))
    g = np.full(H, float(n * steps))  # caller-supplied tally (the adjoint run is row f3)
    _, bits = qmpm.solve_error_bounded(P, g, R, ke32, 0.01, b_min=4, b_max=31)
    _, bits_o = osol.solve_error_bounded(P, g, R, ke32, 0.01, b_min=4, b_max=31)
    assert list(bits) == list(bits_o)
    sch = schemes.from_solution(2, "elastic", R, bits)
    sim = qmpm.Sim(sc.sim, sch, n)
    sim.set_state(dev(st))
    sim.step(steps)
    sq = np.zeros(st.shape, np.float32)
    sim.read_state(vals=sq)
    stats = sim.stats()
    sim.close()
    assert sum(stats.saturations) == 0 and stats.nonfinite == 0
    keq, _ = oracle.aggregates(sc.sim, sq)
    assert abs(keq - ke32) <= 0.02 * abs(ke32), (keq, ke32, list(bits))
