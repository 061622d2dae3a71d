"""Pins of oracle.attention (F4 workload check): closed forms and invariants
of O = softmax(sm_scale Q K^T) V that a dropped term, a wrong sign, a
transposed operand or a softmax over the wrong axis would break."""
import numpy as np

from oracle.attention import attention_rows


def _rand(seed, S=48, D=16):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((S, D)), rng.standard_normal((S, D)), rng.standard_normal((S, D)))


def test_uniform_scores_give_column_mean():
    # identical keys -> all scores of a row equal -> uniform weights -> mean of V
    q, k, v = _rand(1)
    k[:] = k[0]
    out = attention_rows(q, k, v, range(q.shape[0]), 0.3)
    np.testing.assert_allclose(out, np.broadcast_to(v.mean(axis=0), out.shape), rtol=0, atol=1e-12)


def test_zero_scale_gives_column_mean():
    q, k, v = _rand(2, S=37, D=5)   # non-square S x D: a transposed V would not even broadcast
    out = attention_rows(q, k, v, [0, 7, 36], 0.0)
    np.testing.assert_allclose(out, np.broadcast_to(v.mean(axis=0), out.shape), rtol=0, atol=1e-12)


def test_dominant_key_selects_its_value_row():
    q, k, v = _rand(3)
    k = np.zeros_like(k)
    k[11] = 50.0 * q[4] / np.linalg.norm(q[4])     # only key 11 aligns with query 4, by a wide margin
    out = attention_rows(q, k, v, [4], 1.0)
    np.testing.assert_allclose(out[0], v[11], rtol=0, atol=1e-12)


def test_dominant_key_sign_matters():
    # a strongly anti-aligned key gets weight -> 0 (a sign error would select it)
    q, k, v = _rand(4, S=2, D=3)
    k[0] = 30.0 * q[0]
    k[1] = -30.0 * q[0]
    out = attention_rows(q, k, v, [0], 1.0)
    np.testing.assert_allclose(out[0], v[0], rtol=0, atol=1e-12)


def test_joint_key_value_permutation_invariance():
    q, k, v = _rand(5)
    perm = np.random.default_rng(9).permutation(k.shape[0])
    a = attention_rows(q, k, v, range(10), 0.125)
    b = attention_rows(q, k[perm], v[perm], range(10), 0.125)
    np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-13)
    # permuting values alone changes the result (weights are tied to their keys)
    c = attention_rows(q, k, v[perm], range(10), 0.125)
    assert np.abs(a - c).max() > 1e-3


def test_convex_hull_and_two_key_closed_form():
    q, k, v = _rand(6)
    out = attention_rows(q, k, v, range(q.shape[0]), 0.5)
    assert np.all(out <= v.max(axis=0) + 1e-12) and np.all(out >= v.min(axis=0) - 1e-12)
    # two keys: weight of key 0 = 1 / (1 + exp(s1 - s0)), written from the logistic form
    q2, k2, v2 = q[:1], k[:2], v[:2]
    s0, s1 = 0.5 * float(q2[0] @ k2[0]), 0.5 * float(q2[0] @ k2[1])
    w0 = 1.0 / (1.0 + np.exp(s1 - s0))
    np.testing.assert_allclose(attention_rows(q2, k2, v2, [0], 0.5)[0], w0 * v2[0] + (1 - w0) * v2[1],
                               rtol=1e-13, atol=1e-13)


def test_fp16_inputs_converted_exactly():
    q, k, v = (x.astype(np.float16) for x in _rand(7, S=16, D=8))
    a = attention_rows(q, k, v, range(16), 0.25)
    b = attention_rows(q.astype(np.float64), k.astype(np.float64), v.astype(np.float64), range(16), 0.25)
    assert np.array_equal(a, b)
