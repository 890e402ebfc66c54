"""GPU parity of the 3D fixed-corotated stress on hand-picked deformation gradients.

P2G computes (F - R) F^T as B - sqrt(B), B = F F^T, in closed form (eigenvalues of
E = B - I by the trigonometric formula, divided differences of sqrt(1 + mu); DESIGN.md
§5 "Polar decomposition"), not by a polar iteration.  The developed-state tests meet
the F a contact produces; this one aims at the formula's special cases: the identity,
isotropic F = s R (E's eigenvalues coincide: the p -> 0 branch), two equal singular
values (a double eigenvalue), large and tiny strains, simple shear, and a mix.  Every
particle starts at rest (v = 0, C = 0), so after one step the particles' v and C come
from the stress and gravity alone -- a wrong stress shows at full weight.  The fp32
scheme (raw fields) keeps quantisation out; the bar is the P2 bound of
test_gpu_step.py against the fp64 oracle (whose polar factor is a Jacobi SVD).
Inputs are synthetic and seeded; nothing comes from the GPU.
"""
import numpy as np
import pytest

import oracle
from paper_2207_04658_b200 import scenes, schemes
from test_gpu_step import REL, run_gpu_step, scales

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")


def _rot(rng):
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def _family(k, rng):
    R = _rot(rng)
    if k == 0:
        return np.eye(3)
    if k == 1:  # isotropic: B = s^2 I, all of E's eigenvalues equal
        return rng.choice([0.8, 0.95, 1.07, 1.25]) * R
    if k == 2:  # a double singular value
        a, b = rng.uniform(0.8, 1.2, 2)
        return R @ np.diag([a, a, b]) @ _rot(rng).T
    if k == 3:  # large, distinct stretches
        return R @ np.diag(rng.permutation([0.6, 1.0, 1.5])) @ _rot(rng).T
    if k == 4:  # tiny strain (relative accuracy of B - sqrt(B) at small E)
        S = np.eye(3) + 1e-4 * rng.normal(size=(3, 3))
        return R @ (0.5 * (S + S.T))
    if k == 5:  # simple shear
        F = np.eye(3)
        i, j = rng.choice(3, 2, replace=False)
        F[i, j] = rng.uniform(-0.4, 0.4)
        return F
    return R @ (np.eye(3) + 0.1 * rng.normal(size=(3, 3)))  # generic


@pytest.mark.parametrize("seed", [0, 1])
def test_corotated_stress_special_gradients(seed):
    sc = scenes.small_elastic_3d(seed=seed, cube=10)
    sch = schemes.fp32(3)
    st = sc.state().astype(np.float64)
    n = st.shape[0]
    rng = np.random.default_rng(1234 + seed)
    st[:, 3:6] = 0.0   # v
    st[:, 15:24] = 0.0  # C
    for p in range(n):
        st[p, 6:15] = _family(p % 7, rng).reshape(-1)
    assert np.all(np.linalg.det(st[:, 6:15].reshape(-1, 3, 3)) > 0)
    w_in, _ = oracle.encode_state(sch, st.astype(np.float32))
    o_pre, _, _ = oracle.step(sc.sim, sch, w_in, 1, "f64")
    g_pre, _, stats = run_gpu_step(sc, sch, w_in, 1)
    assert stats.nonfinite == 0 and stats.pool_overflow == 0
    s = scales(sc.sim, o_pre, oracle.decode_state(sch, w_in))
    err = np.abs(g_pre.astype(np.float64) - o_pre) / np.maximum(np.abs(o_pre), s)
    worst = err.max(axis=0)
    assert worst.max() <= REL, worst
    # the stress is what moved the particles: v' differs from free fall by far more than the bar
    v_free = np.asarray(sc.sim["gravity"], np.float64) * sc.sim["dt"]
    assert np.abs(o_pre[:, 3:6] - v_free).max() > 100 * REL * s[3]
