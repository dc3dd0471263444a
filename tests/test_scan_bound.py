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
