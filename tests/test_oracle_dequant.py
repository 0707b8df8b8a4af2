"""Pin of the oracle's dequantisation step against exact rational arithmetic (no GPU).

The paper: "we perform integer addition of the offset and the per-vertex value" and
"map the values back to their original floating-point representation".
DESIGN.md reading R11 fixes the map as ONE fused multiply-add in binary32,

    x = fmaf((float)q, Δ_f, g_f),     q = L_c + code (u32),

so the pin is: the oracle's float equals RN32( RN32(q) · Δ_f + g_f ), where RN32 is the
round-to-nearest-even binary32 rounding of an EXACT rational (Python Fraction) and
RN32(q) = q for q < 2^24.  RN32 below is written from the IEEE-754 definition (normal
and subnormal quanta, ties to even, overflow to infinity) and shares nothing with the
oracle.  Inputs straddle 2^24 (where (float)q itself rounds), use negative origins with
cancellation (where a separate multiply and add would round twice), subnormal and huge
products, and random codes at every width of the 24-bit channel.
"""
from fractions import Fraction

import numpy as np
import pytest

from streams import gts_meshlet, pack_meshlets

pytestmark = pytest.mark.filterwarnings("ignore")

_MIN_EXP = -126          # smallest normal exponent of binary32
_QUANTUM_SUB = Fraction(1, 2 ** 149)


def rn32(x: Fraction) -> float:
    """Round an exact rational to the nearest binary32 (ties to even); returns a Python float
    holding that binary32 value exactly (or ±inf)."""
    if x == 0:
        return 0.0
    sign = -1 if x < 0 else 1
    a = -x if x < 0 else x
    # exponent e with 2^e <= a < 2^(e+1)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    elif Fraction(2) ** (e + 1) <= a:
        e += 1
    quantum = _QUANTUM_SUB if e < _MIN_EXP else Fraction(2) ** (e - 23)
    n = a / quantum
    fl = n.numerator // n.denominator
    rem = n - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    r = fl * quantum
    if r >= Fraction(2) ** 128:
        return sign * float("inf")
    return sign * float(r)   # binary32 values are exact in binary64


def test_rn32_self_check():
    """RN32 agrees with numpy's binary32 conversion of binary64 values that are exact
    rationals (a check of the helper only; numpy is not the oracle)."""
    rng = np.random.default_rng(7)
    vals = np.concatenate([rng.normal(size=2000) * 10.0 ** rng.integers(-45, 38, 2000),
                           [1.5 * 2.0 ** -149, 2.5 * 2.0 ** -149, 3.4e38, 3.5e38, 2.0 ** 24 + 1, 2.0 ** 24 + 3]])
    for v in vals:
        want = np.float32(v)   # numpy rounds binary64 -> binary32 RNE
        assert rn32(Fraction(float(v))) == float(want) or (np.isinf(want) and np.isinf(rn32(Fraction(float(v))))), v


def _cases():
    """(L, code, Δ, g) tuples: one object per (Δ, g), one meshlet per (object, L)."""
    f32 = lambda v: float(np.float32(v))
    deltas = [1.0, f32(1e-3), f32(3.0517578e-05), f32(1.4e-40), f32(7e-46 * 2 ** 10), f32(1e30), f32(0.1)]
    origins = [0.0, -1.5, f32(123.456), f32(-3.0e7), f32(-1e-38)]
    Ls = [0, (1 << 24) - 300, 1 << 24, (1 << 24) + 1, (1 << 27) + 5, (1 << 31) - 1000, (1 << 32) - (1 << 24) - 1]
    return deltas, origins, Ls


def test_dequant_is_single_rounding_of_exact_rational(orc):
    """P:490-494 under reading R11: oracle float == RN32(RN32(q)·Δ + g) for every vertex."""
    deltas, origins, Ls = _cases()
    rng = np.random.default_rng(11)
    objs = [(d, g) for d in deltas for g in origins]
    # cancellation objects: g = -RN32(q0·Δ) for a q0 inside the meshlet range, so the exact
    # result is tiny and a separately rounded product would be off by many ulps
    canc = []
    for L in Ls[:5]:
        for d in (f32 for f32 in (float(np.float32(1e-3)), float(np.float32(0.1)))):
            q0 = L + 1000
            canc.append((d, -rn32(Fraction(rn32(Fraction(q0))) * Fraction(d))))
    objs += canc
    V = 256
    meshlets, Lall, obj, codes = [], [], [], []
    for oi in range(len(objs)):
        for L in Ls:
            meshlets.append(gts_meshlet(V, [], []))
            Lall.append(L)
            obj.append(oi)
            c = rng.integers(0, 1 << 24, V).astype(np.uint32)
            c[:6] = [0, 1, (1 << 24) - 1, 1000, 999, 1001]    # edges, and q0 of the cancellation objects
            codes.append(c)
    delta = np.array([d for d, _ in objs], np.float32)
    origin = np.array([g for _, g in objs], np.float32)
    blob = pack_meshlets(orc, 1, meshlets, n=1, bits=(24,), codes=np.concatenate(codes), L=np.array(Lall, np.uint32),
                         delta=delta, origin=origin, obj=obj, vmax=256, tmax=256)
    err, errs, idx, q, f = orc.decode(blob)
    assert err == 0
    q = q.astype(np.int64)
    k = 0
    bad = []
    checked_above = 0
    for mi, (L, oi) in enumerate(zip(Lall, obj)):
        d, g = Fraction(float(delta[oi])), Fraction(float(origin[oi]))
        for v in range(V):
            qq = L + int(codes[mi][v])
            assert q[k] == qq                        # q = L + code
            qf = Fraction(rn32(Fraction(qq)))        # (float)q: exact below 2^24, rounded above
            want = rn32(qf * d + g)
            got = float(f[k])
            if not (got == want or (np.isinf(want) and got == want)):
                bad.append((qq, float(delta[oi]), float(origin[oi]), got, want))
            checked_above += qq >= (1 << 24)
            k += 1
    assert not bad, bad[:5]
    assert checked_above > 10000


def test_dequant_pin_detects_double_rounding(orc):
    """The cancellation cases above are sensitive: RN32(RN32(qΔ) + g) (a separate product
    and sum) differs from the single rounding for some of them, so a mul+add oracle would
    fail the pin (self-check of the test's power)."""
    d = float(np.float32(0.1))
    diffs = 0
    for q in range((1 << 24) - 3000, (1 << 24) - 2000):
        g = -rn32(Fraction(q - 7) * Fraction(d))
        one = rn32(Fraction(q) * Fraction(d) + Fraction(g))
        two = rn32(Fraction(rn32(Fraction(q) * Fraction(d))) + Fraction(g))
        diffs += one != two
    assert diffs > 100
