"""The oracle against the worked examples the paper / its specification print
(tests/golden/paper_examples.json, each entry with its citation)."""
import json
import os

import numpy as np

import oracle
from test_oracle_codec import fixed_scheme
from test_oracle_mpm import particle, sim2d

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def test_codec_round_examples():
    for ex in GOLDEN["codec_round"]:
        s = fixed_scheme([ex["frac_bits"]], [ex["range"]], rounding="rne")
        w, cnt = oracle.encode(s, np.array([[ex["v"]]], np.float32))
        assert int(w[0, 0]) == ex["u"], ex["cite"]
        assert float(oracle.decode(s, w)[0, 0]) == ex["decoded"], ex["cite"]
        assert int(cnt[0]) == ex["saturated"], ex["cite"]


def test_layout_examples():
    for ex in GOLDEN["layout"]:
        s = fixed_scheme([w - 1 for w in ex["widths"]], [1.0] * len(ex["widths"]))
        offs, W, bits = oracle.layout(s)
        assert list(offs) == ex["offsets"] and W == ex["words"] and bits == ex["bits"], ex["cite"]


def test_cross_word_examples():
    L = oracle.lib()
    for ex in GOLDEN["cross_word"]:
        rec = np.array(ex["words"], np.uint32)
        assert L.oracle_get_bits(rec.ctypes.data, ex["offset"], ex["width"]) == ex["value"], ex["cite"]


def test_drift_example():
    for ex in GOLDEN["drift"]:
        b, R = 16, 2.0 ** 16  # Delta = 1 (wide type, reading Q7)
        s_rne = fixed_scheme([b], [R], rounding="rne")
        s_dit = fixed_scheme([b], [R], rounding="dither")
        n = ex["trials"]
        y_rne = np.zeros((1, 1), np.float32)
        y_dit = np.zeros((n, 1), np.float32)
        keys = np.arange(n, dtype=np.uint32) * np.uint32(7919)
        inc = np.float32(ex["increment_deltas"])
        for t in range(1, ex["steps"] + 1):
            y_rne = oracle.decode(s_rne, oracle.encode(s_rne, y_rne + inc)[0])
            y_dit = oracle.decode(s_dit, oracle.encode(s_dit, y_dit + inc, keys=keys, step=t)[0])
        assert float(y_rne[0, 0]) == ex["undithered_deltas"], ex["cite"]
        assert abs(float(y_dit.mean()) - ex["dithered_mean_deltas"]) < ex["dithered_tol_deltas"], ex["cite"]


def test_dither_probability_example():
    for ex in GOLDEN["dither_probability"]:
        s = fixed_scheme([16], [2.0 ** 16], rounding="dither")  # Delta = 1, so t = v
        n = 200_000
        keys = np.arange(n, dtype=np.uint32)
        w, _ = oracle.encode(s, np.full((n, 1), ex["t"], np.float32), keys=keys, step=1)
        up = float(np.mean(oracle.decode(s, w)[:, 0] > ex["t"]))
        assert abs(up - ex["p_up"]) < 4 * np.sqrt(ex["p_up"] * (1 - ex["p_up"]) / n), ex["cite"]


def test_bspline_examples():
    s = sim2d()
    for ex in GOLDEN["bspline"]:
        x = (5.0 + ex["fx"]) * s["dx"]  # base = floor(x/dx - 1/2) = 5, fx = x/dx - 5
        st = particle(2, [x, x])[None]
        grid, origin, gsize, _ = oracle.p2g(s, st)
        m = grid[..., 0, 0] / (s["p_rho"] * s["p_vol"])
        w = np.array(ex["w"])
        np.testing.assert_allclose(m, np.outer(w, w), rtol=0, atol=1e-15, err_msg=ex["cite"])
