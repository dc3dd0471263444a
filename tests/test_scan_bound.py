"""The screened scan's error bound (scpl_stats.cu: kScanDelta), checked in exact arithmetic.

The screening kernel computes the variance as fma(-m, m, RN(Q*rn)) with m = RN(S*rn),
rn = RN(1/n); the reference (buffering.py:174-176) as RN(RN(Q/n) - RN(RN(S/n)^2)).  Both are
evaluated here with exact rationals and one correct rounding per operation (float(Fraction)
rounds to nearest), over energies drawn from the reference's motion-energy values, and the
difference must stay under the kernel's kScanDelta = 2e-10 (derived: 14.2 u X <= 1.03e-10).
The std bound min(sqrt(delta), delta / std~) is checked on the same samples."""
import math
from fractions import Fraction

import numpy as np

KSCAN_DELTA = 2.0e-10


def _rn(x: Fraction) -> float:
    return float(x)  # correctly rounded to nearest even


def _energies(rng, n, wm=0.6, wg=0.4, extreme=False):
    d = rng.integers(0, 256, n) if not extreme else rng.integers(250, 256, n)
    g = rng.integers(0, 256, n) if not extreme else rng.integers(250, 256, n)
    e = np.minimum(np.float64(wm) * d + np.float64(wg) * g, 255.0)  # fl(fl(wm d) + fl(wg g)), clamped
    return [float(x) for x in e]


def _sums(es):
    S = Q = 0.0
    for e in es:  # stream order, separate roundings (buffering.py:116-117)
        S = S + e
        Q = Q + e * e
    return S, Q


def test_screened_variance_within_bound():
    rng = np.random.default_rng(1234)
    worst = 0.0
    for trial in range(3000):
        n = int(rng.integers(1, 65))
        es = _energies(rng, n, extreme=trial % 3 == 0)
        if trial % 7 == 0:  # near-constant pixels: variance ~ 0, the cancellation-heavy case
            es = [es[0]] * n
        S, Q = _sums(es)
        # reference
        m_r = S / n
        var_r = (Q / n) - (m_r * m_r)
        # screened (exact rationals, one rounding per op; the fma rounds once)
        rn = _rn(Fraction(1) / n)
        m_a = _rn(Fraction(S) * Fraction(rn))
        v1 = _rn(Fraction(Q) * Fraction(rn))
        var_a = _rn(Fraction(v1) - Fraction(m_a) ** 2)
        diff = abs(var_a - var_r)
        worst = max(worst, diff)
        assert diff <= KSCAN_DELTA, (n, S, Q, var_a, var_r)
        sd_r = math.sqrt(max(var_r, 0.0))
        v = max(var_a, 1e-30)
        sd_a = v / math.sqrt(v)
        bound = min(math.sqrt(KSCAN_DELTA), KSCAN_DELTA / math.sqrt(v))
        assert abs(sd_a - sd_r) <= bound * (1 + 1e-6) + 1e-15 + 1e-12 * sd_r, (var_a, var_r, sd_a, sd_r)
    assert worst < 1.03e-10 * 1.01  # the derivation's constant holds on these samples


def _f64_f32_floor(x):
    """scpl_stats.cu f64_f32_floor in numpy: max(var, ~1e-30) on the high word, exponent re-bias,
    funnel shift by 3 (truncation to f32)."""
    u = np.asarray(x, dtype=np.float64).view(np.uint64)
    hi = (u >> np.uint64(32)).astype(np.int64)
    hi = np.where(hi >= 2 ** 31, hi - 2 ** 32, hi)  # signed high word: negatives sort below
    lo = (u & np.uint64(0xFFFFFFFF)).astype(np.int64)
    hi = np.maximum(hi, 0x39B4484B)
    bits = ((((hi - 0x38000000) << 3) & 0xFFFFFFFF) | (lo >> 29)).astype(np.uint32)
    return bits.view(np.float32)


def test_screen_float_conversion_is_a_floor_within_2pow23():
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.uniform(0.0, 65025.0, 200000), 10.0 ** rng.uniform(-29.9, 4.8, 200000),
                        np.array([1e-30, 65025.0, 0.25, 1.0, 255.0 ** 2])])
    f = _f64_f32_floor(x).astype(np.float64)
    assert np.all(f <= x) and np.all(f > 0)
    assert np.max((x - f) / x) < 2.0 ** -23
    # zero, negative and tiny variances clamp to about 1e-30 (the kernel's floor), never NaN / inf
    low = _f64_f32_floor(np.array([0.0, -0.0, -1.0, -1e-300, 1e-40, 1e-31])).astype(np.float64)
    assert np.all((low >= 0.99e-30) & (low < 2.1e-30))


def test_clamp_free_energy_condition():
    """screen_noclamp / uniform_noclamp: with non-negative weights and fl(fl(255 wm) + fl(255 wg))
    <= 255 no motion energy exceeds 255, so min(e, 255) is the identity on all 65536 codes."""
    d, g = np.meshgrid(np.arange(256, dtype=np.float64), np.arange(256, dtype=np.float64), indexing="ij")
    rng = np.random.default_rng(11)
    cases = [(0.6, 0.4), (0.5, 0.5), (1.0, 0.0), (0.0, 1.0), (0.3, 0.7)]
    cases += [tuple(rng.uniform(0, 1, 2)) for _ in range(200)]
    held = 0
    for wm, wg in cases:
        wm, wg = np.float64(wm), np.float64(wg)
        cond = (wm * 255.0) + (wg * 255.0) <= 255.0
        e = (wm * d) + (wg * g)  # separate roundings, as energy.py:86 computes it
        if cond:
            held += 1
            assert e.max() <= 255.0 and np.array_equal(np.minimum(e, 255.0), e), (wm, wg)
            assert not np.signbit(e).any()
    assert held >= 5 and (np.float64(0.6) * 255.0) + (np.float64(0.4) * 255.0) <= 255.0


def test_byte_to_double_on_the_fp64_pipe():
    """u8_f64: the double with high word 0x43300000 and low word k is 2^52 + k; minus 2^52 is k."""
    k = np.arange(256, dtype=np.uint64)
    v = ((np.uint64(0x43300000) << np.uint64(32)) | k).view(np.float64) - 4503599627370496.0
    assert np.array_equal(v, np.arange(256, dtype=np.float64))
