"""GPU parity of the quantized MLS-MPM step (P2, P3) through the C ABI.

P2 (single step, BASELINE north_star: "within 1e-5 relative (fp32)"): identical
packed input words (qmpm_set_words) -> one step -> the GPU's pre-encode fp32 state
(QMPM_DEBUG_PREENCODE) vs the fp64 oracle, per component:
    |g - o| <= 1e-5 * max(|o|, s_h)
with the conditioning-aware scale s_h of SURVEY §8(c) P2: x -> domain extent 1,
v -> max(RMS v, |g| dt), C -> 4/dx * s_v, F and J -> 1.  Then P1 on those floats:
the GPU's stored words must equal the oracle codec applied to the GPU's own
pre-encode floats (same content keys, same step) BIT-EXACTLY, and the stored codes
may differ from the oracle's own codes only by rounding-boundary flips (fp32 atomic
order; reading Q22).
P3 (100 steps): kinetic energy and centre of mass within 1e-3 relative.
"""
import numpy as np
import pytest

import oracle
from paper_2207_04658_b200 import qmpm, scenes, schemes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

REL = 1e-5


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def scales(sim, o, inp=None):
    """Conditioning-aware scale per state scalar (DESIGN.md §5 "P2 tolerance").
    fp32 summation error is bounded by eps * sum|terms|, so v is measured against the
    magnitude of the P2G momentum terms in velocity units: |v|, |g| dt, |C| dx (APIC
    term) and dt 4 (2 mu + d lambda) |F - I| / (rho dx) (stress term; fluid: E |J - 1|),
    RMS over particles of the INPUT state.  C is a cancelling sum of node velocities
    (C' = 4/dx sum w v_i (x) (i - fx)), so its scale is 4/dx * s_v."""
    d = sim["dim"]
    ns = o.shape[1]
    s = np.ones(ns)
    s[:d] = 1.0
    g = np.linalg.norm(sim["gravity"])
    terms = [float(np.sqrt(np.mean(o[:, d:2 * d] ** 2))), g * sim["dt"], 1e-12]
    if inp is not None:
        inp = inp.astype(np.float64)
        fluid = sim["material"] == "fluid"
        C = inp[:, -d * d:]
        terms.append(float(np.sqrt(np.mean(np.sum(C ** 2, 1)))) * sim["dx"])
        E, nu = sim["E"], sim["nu"]
        if fluid:
            strain = np.abs(inp[:, 2 * d] - 1.0)
            k = E
        else:
            F = inp[:, 2 * d:2 * d + d * d]
            strain = np.sqrt(np.sum((F - np.eye(d).reshape(-1)) ** 2, 1))
            mu = E / (2 * (1 + nu))
            la = E * nu / ((1 + nu) * (1 - 2 * nu))
            k = 2 * mu + d * la
        terms.append(float(np.sqrt(np.mean(strain ** 2))) * sim["dt"] * 4 * k / (sim["p_rho"] * sim["dx"]))
    sv = max(terms)
    s[d:2 * d] = sv
    s[-d * d:] = 4.0 / sim["dx"] * sv
    return s


def run_gpu_step(sc, sch, words_in, step_index, n_steps=1, pool_blocks=0):
    n = words_in.shape[0]
    sim = qmpm.Sim(sc.sim, sch, n, flags=qmpm.TRACK_IDS | qmpm.DEBUG_PREENCODE, pool_blocks=pool_blocks)
    sim.set_words(dev(words_in), step_index - 1)
    sim.step(n_steps)
    ns = sim.n_scalars
    pre = np.zeros((n, ns), np.float32)
    words = np.zeros_like(words_in)
    ids = np.zeros(n, np.uint32)
    sim.read_state(words=words, ids=ids)
    sim.read_debug(pre)
    st = sim.stats()
    sim.close()
    inv = np.argsort(ids)
    return pre[inv], words[inv], st


CASES = {
    "c1_2d_x16": (scenes.c1, schemes.x16, 30),
    "s3_3d_e0.1": (scenes.small_elastic_3d, schemes.e01, 20),
    "s3_3d_e0.01": (scenes.small_elastic_3d, schemes.e001, 20),
    "s3_3d_fp32": (scenes.small_elastic_3d, lambda: schemes.fp32(3), 20),
    "s4_3d_fluid_f2": (scenes.small_fluid_3d, schemes.f2, 20),
    "s4_3d_fluid_se2": (scenes.small_fluid_3d, schemes.se2, 20),
    # no field straddles a word (the bit struct's rule; T-bitpack-perf analogue)
    "s3_3d_e0.01_nostraddle": (scenes.small_elastic_3d, lambda: schemes.with_layout(schemes.e001(), "nostraddle"), 20),
    "s4_3d_fluid_f2_nostraddle": (scenes.small_fluid_3d, lambda: schemes.with_layout(schemes.f2(), "nostraddle"), 20),
    # a 32^3 grid: 512 blocks, one scan tile, so the step's sort front is the fused
    # one-CTA k_sort_small (C1 takes it in 2D)
    "s4_3d_fluid_f2_res32": (lambda: scenes.small_fluid_3d(res=32, n_target=20_000), schemes.f2, 20),
}


@pytest.mark.parametrize("case", list(CASES))
def test_single_step_parity(case):
    mk_scene, mk_scheme, warm = CASES[case]
    sc, sch = mk_scene(), mk_scheme()
    w0, _ = oracle.encode_state(sch, sc.state())
    # warm-up by the ORACLE so F != I and C != 0 (inputs never come from the GPU)
    w_in, _ = oracle.run(sc.sim, sch, w0, 1, warm)
    t = warm + 1
    o_pre, o_words, _ = oracle.step(sc.sim, sch, w_in, t, "f64")
    g_pre, g_words, st = run_gpu_step(sc, sch, w_in, t)
    assert st.pool_overflow == 0 and st.nonfinite == 0
    s = scales(sc.sim, o_pre, oracle.decode_state(sch, w_in))
    err = np.abs(g_pre.astype(np.float64) - o_pre) / np.maximum(np.abs(o_pre), s)
    worst = err.max(axis=0)
    assert worst.max() <= REL, (case, worst)
    # P1 on the GPU's own pre-encode floats: same keys (content of the input record), same step
    keys = np.array([oracle.particle_key(sch, w_in[i]) for i in range(w_in.shape[0])], np.uint32)
    w_p1, _ = oracle.encode_state(sch, g_pre, step=t, keys=keys)
    assert np.array_equal(g_words, w_p1)
    # stored codes vs the oracle's own codes: only rounding-boundary flips
    dg = oracle.decode_state(sch, g_words).astype(np.float64)
    do = oracle.decode_state(sch, o_words).astype(np.float64)
    nfld = len(sch["fields"])
    deltas = np.ones(dg.shape[1])
    for f in sch["fields"]:
        if f["kind"] == "fixed":
            idx = oracle.scalar_index(f["attr"], f["comp"], sch["dim"], sch["material"])
            deltas[idx] = f["range"] * 2.0 ** -f["frac_bits"]
    fixed = np.array([f["kind"] == "fixed" for f in sorted(
        sch["fields"], key=lambda f: oracle.scalar_index(f["attr"], f["comp"], sch["dim"], sch["material"]))])
    if fixed.any():
        code_diff = np.abs(dg - do)[:, fixed] / deltas[fixed]
        assert code_diff.max() <= 1.0 + 1e-6
        assert np.mean(code_diff > 0.5) <= 2e-3, np.mean(code_diff > 0.5)
    assert nfld == dg.shape[1]


@pytest.mark.parametrize("case", ["c1_2d_x16", "s3_3d_e0.1", "s4_3d_fluid_f2"])
def test_fp32_oracle_agrees_too(case):
    """The fp32 oracle instantiation is a second comparator: each fp32 implementation
    is within REL of the fp64 truth, so the two differ by at most 2 REL (triangle
    inequality on the same scales)."""
    mk_scene, mk_scheme, warm = CASES[case]
    sc, sch = mk_scene(), mk_scheme()
    w0, _ = oracle.encode_state(sch, sc.state())
    w_in, _ = oracle.run(sc.sim, sch, w0, 1, 5)
    o32, _, _ = oracle.step(sc.sim, sch, w_in, 6, "f32")
    o64, _, _ = oracle.step(sc.sim, sch, w_in, 6, "f64")
    g_pre, _, _ = run_gpu_step(sc, sch, w_in, 6)
    s = scales(sc.sim, o64, oracle.decode_state(sch, w_in))
    den = np.maximum(np.abs(o64), s)
    assert (np.abs(o32 - o64) / den).max() <= REL
    assert (np.abs(g_pre.astype(np.float64) - o64) / den).max() <= REL
    assert (np.abs(g_pre.astype(np.float64) - o32) / den).max() <= 2 * REL


def aggregates(sim, st):
    return oracle.aggregates(sim, st)


@pytest.mark.parametrize("case,steps", [("c1_2d_x16", 100), ("s3_3d_e0.1", 100), ("s4_3d_fluid_f2", 100),
                                        ("s4_3d_fluid_se2", 100)])
def test_100_step_aggregates(case, steps):
    """P3: KE and COM after 100 steps within 1e-3 relative (GPU vs fp64 oracle)."""
    mk_scene, mk_scheme, _ = CASES[case]
    sc, sch = mk_scene(), mk_scheme()
    st0 = sc.state()
    w0, _ = oracle.encode_state(sch, st0)
    w_o, _ = oracle.run(sc.sim, sch, w0, 1, steps)
    so = oracle.decode_state(sch, w_o)
    sim = qmpm.Sim(sc.sim, sch, st0.shape[0])
    sim.set_state(dev(st0))
    sim.step(steps)
    sg = np.zeros(st0.shape, np.float32)
    sim.read_state(vals=sg)
    stats = sim.stats()
    sim.close()
    assert stats.step == steps
    ke_o, com_o = aggregates(sc.sim, so)
    ke_g, com_g = aggregates(sc.sim, sg)
    assert abs(ke_g - ke_o) <= 1e-3 * abs(ke_o), (ke_g, ke_o)
    assert np.all(np.abs(com_g - com_o) <= 1e-3 * np.abs(com_o)), (com_g, com_o)


def test_ragged_edge_cases():
    """n = 0, a single particle, and n = 33 (one full warp + 1) all step cleanly and match."""
    sc = scenes.small_elastic_3d()
    sch = schemes.e01()
    sim = qmpm.Sim(sc.sim, sch, 64, flags=qmpm.TRACK_IDS | qmpm.DEBUG_PREENCODE)
    sim.set_state(dev(sc.state()[:0]))
    sim.step(3)
    assert sim.stats().n_particles == 0
    for n in (1, 33):
        st = sc.state()[:n]
        w, _ = oracle.encode_state(sch, st)
        o_pre, o_words, _ = oracle.step(sc.sim, sch, w, 1)
        sim.set_words(dev(w), 0)
        sim.step(1)
        pre = np.zeros((n, 24), np.float32)
        ids = np.zeros(n, np.uint32)
        sim.read_state(ids=ids)
        sim.read_debug(pre)
        pre = pre[np.argsort(ids)]
        s = scales(sc.sim, o_pre)
        assert (np.abs(pre - o_pre) / np.maximum(np.abs(o_pre), s)).max() <= REL
    sim.close()


def test_out_of_domain_counted_and_clamped():
    """Reading Q14: a particle whose base leaves [0, n-3] is clamped and counted."""
    sc = scenes.small_elastic_3d()
    sch = schemes.fp32(3)
    st = sc.state()[:40].copy()
    st[:5, 0] = 0.2 / 64  # base = floor(0.2 - 0.5) = -1 -> clamped to 0
    w, _ = oracle.encode_state(sch, st)
    o_pre, _, oc = oracle.step(sc.sim, sch, w, 1)
    g_pre, _, gst = run_gpu_step(sc, sch, w, 1)
    assert oc[193] == 5 and gst.out_of_domain == 5
    s = scales(sc.sim, o_pre)
    assert (np.abs(g_pre - o_pre) / np.maximum(np.abs(o_pre), s)).max() <= REL


def test_pool_overflow_reported():
    sc = scenes.small_elastic_3d()
    sch = schemes.e01()
    st = sc.state()
    sim = qmpm.Sim(sc.sim, sch, st.shape[0], pool_blocks=4)
    sim.set_state(dev(st))
    sim.step(1)
    with pytest.raises(qmpm.QmpmError) as e:
        sim.read_state(vals=np.zeros(st.shape, np.float32))
    assert e.value.code == 8
    assert sim.stats().pool_overflow == 1
    sim.close()


def test_resume_from_words_is_consistent():
    """set_words(words, t) resumes: the next step's dither uses step t+1 (reading Q5)."""
    sc = scenes.c1()
    sch = schemes.x16()
    w0, _ = oracle.encode_state(sch, sc.state())
    w5, _ = oracle.run(sc.sim, sch, w0, 1, 5)
    o_pre, o_w, _ = oracle.step(sc.sim, sch, w5, 6)
    g_pre, g_w, _ = run_gpu_step(sc, sch, w5, 6)
    keys = np.array([oracle.particle_key(sch, w5[i]) for i in range(w5.shape[0])], np.uint32)
    assert np.array_equal(g_w, oracle.encode_state(sch, g_pre, step=6, keys=keys)[0])


def test_round_counters_match_oracle_on_identical_floats():
    """Round-up / round-down / saturation counters (T-dither-eff) equal
    the oracle codec's on the GPU's own pre-encode floats."""
    sc = scenes.c1()
    sch = schemes.x16()
    w0, _ = oracle.encode_state(sch, sc.state())
    w_in, _ = oracle.run(sc.sim, sch, w0, 1, 10)
    g_pre, _, st = run_gpu_step(sc, sch, w_in, 11)
    keys = np.array([oracle.particle_key(sch, w_in[i]) for i in range(w_in.shape[0])], np.uint32)
    _, c = oracle.encode_state(sch, g_pre, step=11, keys=keys)
    nf = len(sch["fields"])
    assert list(st.round_up)[:nf] == list(c[64:64 + nf])
    assert list(st.round_down)[:nf] == list(c[128:128 + nf])
    assert list(st.saturations)[:nf] == list(c[:nf])


@pytest.mark.parametrize("case", ["s3_3d_e0.01", "s4_3d_fluid_f2", "c1_2d_x16"])
def test_p2g_short_segments(case, monkeypatch):
    """Short P2G segments (many groups straddling levels, so lanes sharing a cell take
    turns in the flush) and the level cap (cells with more than kSegLev segments, whose
    last segment takes the rest) meet the same P2 bar: the step kernels are
    re-specialised with a segment length of 2 particles."""
    monkeypatch.setenv("QMPM_JIT_OPTS", "-DQMPM_SEG_L=2 -DQMPM_SEG_LMIN=2")
    mk_scene, mk_scheme, warm = CASES[case]
    sc, sch = mk_scene(), mk_scheme()
    w0, _ = oracle.encode_state(sch, sc.state())
    w_in, _ = oracle.run(sc.sim, sch, w0, 1, 3)
    o_pre, _, _ = oracle.step(sc.sim, sch, w_in, 4, "f64")
    g_pre, g_words, st = run_gpu_step(sc, sch, w_in, 4)
    s = scales(sc.sim, o_pre, oracle.decode_state(sch, w_in))
    err = np.abs(g_pre.astype(np.float64) - o_pre) / np.maximum(np.abs(o_pre), s)
    assert err.max() <= REL, err.max(axis=0)
    keys = np.array([oracle.particle_key(sch, w_in[i]) for i in range(w_in.shape[0])], np.uint32)
    assert np.array_equal(g_words, oracle.encode_state(sch, g_pre, step=4, keys=keys)[0])


@pytest.mark.parametrize("rounding", ["dither", "rne"])
def test_saturating_step_matches_codec(rounding):
    """A v range far below the velocities forces the G2P re-encode's rare (exact,
    saturating) path: the stored words and the saturation / round counters still equal
    the oracle codec's on the GPU's pre-encode floats."""
    sc = scenes.c1()
    sch = schemes.with_rounding(schemes.x16(v_range=2.0 ** -6), rounding)
    w0, _ = oracle.encode_state(sch, sc.state())
    w_in, _ = oracle.run(sc.sim, sch, w0, 1, 40)
    g_pre, g_words, st = run_gpu_step(sc, sch, w_in, 41)
    keys = np.array([oracle.particle_key(sch, w_in[i]) for i in range(w_in.shape[0])], np.uint32)
    w_ref, c = oracle.encode_state(sch, g_pre, step=41, keys=keys)
    assert np.array_equal(g_words, w_ref)
    nf = len(sch["fields"])
    assert sum(c[:nf]) > 0  # the case really saturates
    assert list(st.saturations)[:nf] == list(c[:nf])
    assert list(st.round_up)[:nf] == list(c[64:64 + nf])
    assert list(st.round_down)[:nf] == list(c[128:128 + nf])
