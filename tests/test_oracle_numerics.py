"""Pins for oracle/numerics.py and oracle/model.py against worked examples, closed forms
and library routines (never against a re-typed copy of the oracle's own formula)."""
import json
import math
import os

import numpy as np
import pytest
import torch

import synth
from oracle.model import Model, ModelConfig
from oracle.numerics import log_softmax, rms_norm, rope_rotate_half, softmax_masked


def _num(x):
    if isinstance(x, str):
        return {"ln2": math.log(2), "ln3": math.log(3), "1/3": 1 / 3, "2/3": 2 / 3}[x]
    return float(x)


@pytest.fixture(scope="module")
def ex(golden_dir):
    return json.load(open(os.path.join(golden_dir, "spec_worked_examples.json")))


def test_softmax_masked_spec_examples(ex):
    for case in ex["softmax_masked"]:
        s = np.array([_num(v) for v in case["scores"]])
        out = softmax_masked(s, np.array(case["allow"]))
        np.testing.assert_allclose(out, [_num(v) for v in case["out"]], atol=1e-15)
        assert np.all(out[~np.array(case["allow"])] == 0.0)  # exactly zero


def test_softmax_all_masked_raises():
    with pytest.raises(ValueError):
        softmax_masked(np.zeros(3), np.zeros(3, bool))


def test_attention_scores_spec(ex):
    c = ex["attention_scores"]
    out = softmax_masked(np.array([_num(v) for v in c["scores"]]), np.ones(2, bool))
    np.testing.assert_allclose(out, c["out"], atol=1e-15)


def test_softmax_shift_invariance():
    s = synth.normal(1, 1, (17,))
    allow = synth.uniform01(1, 2, 17) < 0.6
    allow[0] = True
    np.testing.assert_allclose(softmax_masked(s, allow), softmax_masked(s + 123.0, allow), atol=1e-14)


def test_rope_examples(ex):
    c = ex["rope"]
    np.testing.assert_allclose(rope_rotate_half(np.array(c["vec"], float), c["pos"], 10000.0),
                               c["out"], atol=1e-15)
    v = synth.normal(3, 1, (4, 16))
    np.testing.assert_array_equal(rope_rotate_half(v, 0, 10000.0), v)  # zero angle


def test_rope_isometry_and_composition():
    v = synth.normal(4, 1, (3, 32))
    r = rope_rotate_half(v, 37, 500000.0)
    np.testing.assert_allclose(np.linalg.norm(r, axis=-1), np.linalg.norm(v, axis=-1), rtol=1e-13)
    np.testing.assert_allclose(rope_rotate_half(rope_rotate_half(v, 11, 1e4), 26, 1e4),
                               rope_rotate_half(v, 37, 1e4), atol=1e-12)


def test_rope_matches_complex_rotation():
    # closed form: pair (x_i, x_{i+D/2}) is the complex number x_i + j x_{i+D/2} times e^{j pos theta_i}
    D, pos, base = 16, 5, 10000.0
    v = synth.normal(5, 1, (D,))
    z = (v[: D // 2] + 1j * v[D // 2:]) * np.exp(1j * pos * base ** (-2.0 * np.arange(D // 2) / D))
    np.testing.assert_allclose(rope_rotate_half(v, pos, base), np.concatenate([z.real, z.imag]), atol=1e-14)


def test_rms_norm_examples(ex):
    for c in ex["rms_norm"]:
        np.testing.assert_allclose(rms_norm(np.array(c["v"], float), np.array(c["g"], float), c["eps"]),
                                   c["out"], atol=1e-15)


def test_log_softmax_vs_torch():
    x = synth.normal(6, 1, (300,)) * 5
    np.testing.assert_allclose(log_softmax(x), torch.log_softmax(torch.from_numpy(x), 0).numpy(), atol=1e-13)


# ---------------------------------------------------------------------------------------
def _model(seed=0, Hkv=4, kappa=4.0, V=256, L=2):
    cfg = ModelConfig(L=L, d=64, Hq=4, Hkv=Hkv, D=16, ffn=256, V=V, kappa=kappa)
    w = synth.tiny_weights(seed, cfg.L, cfg.d, cfg.Hq, cfg.Hkv, cfg.D, cfg.ffn, cfg.V)
    return Model(w, cfg)


def test_attend_vs_torch_sdpa():
    m = _model()
    q = synth.normal(7, 1, (4, 16))
    K = synth.normal(7, 2, (9, 4, 16))
    V = synth.normal(7, 3, (9, 4, 16))
    o = m.attend(q, K, V)
    tq = torch.from_numpy(q)[:, None, :]               # [H][1][D]
    tk = torch.from_numpy(K).permute(1, 0, 2)          # [H][n][D]
    tv = torch.from_numpy(V).permute(1, 0, 2)
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv)[:, 0, :].numpy()
    np.testing.assert_allclose(o, ref, atol=1e-13)


@pytest.mark.parametrize("window", [0, 3])
def test_incremental_equals_full_recompute(window):
    """incremental decode == from-scratch causal forward (<= 1e-9)."""
    m = _model(seed=1)
    toks = [int(x) for x in synth.randint(9, 1, 6, 256)]
    full = m.forward_full_causal(toks, window=window)
    cache = [[] for _ in range(m.cfg.L)]
    for p, tk in enumerate(toks):
        def ctx(l, k, v, p=p):
            cache[l].append((k, v))
            lo = 0 if window <= 0 else max(0, p - window + 1)
            rows = cache[l][lo: p + 1]
            return np.stack([r[0] for r in rows]), np.stack([r[1] for r in rows])
        lp = m.forward(tk, p, ctx)
        np.testing.assert_allclose(lp, full[p], atol=1e-9)


def test_gqa_single_kv_head_equals_broadcast_mha():
    """Hkv=1 == MHA whose K/V projections are the single head repeated."""
    g = _model(seed=2, Hkv=1)
    wq = synth.tiny_weights(2, 2, 64, 4, 1, 16, 256, 256)
    w_mha = dict(wq)
    w_mha["layers"] = []
    for lw in wq["layers"]:
        lw2 = dict(lw)
        lw2["wk"] = np.tile(lw["wk"], (1, 4))
        lw2["wv"] = np.tile(lw["wv"], (1, 4))
        w_mha["layers"].append(lw2)
    mha = Model(w_mha, ModelConfig(Hkv=4))
    toks = [5, 17, 200, 3]
    a = g.forward_full_causal(toks)
    b = mha.forward_full_causal(toks)
    np.testing.assert_allclose(a, b, atol=1e-12)


def test_weights_bounds_and_determinism():
    w1 = synth.tiny_weights(5, 2, 64, 4, 4, 16, 256, 256)
    w2 = synth.tiny_weights(5, 2, 64, 4, 4, 16, 256, 256)
    w3 = synth.tiny_weights(6, 2, 64, 4, 4, 16, 256, 256)
    assert np.array_equal(w1["layers"][1]["wd"], w2["layers"][1]["wd"])
    assert not np.array_equal(w1["layers"][1]["wd"], w3["layers"][1]["wd"])
    assert np.abs(w1["layers"][0]["wq"]).max() <= 1 / 8  # fan_in 64
