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
    # against the oracle's pre-encode state of the same step (P2 tolerance of the values)
    w = np.zeros((n, sim.W), np.uint32)
    sim.read_state(words=w)
    sim.close()


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
