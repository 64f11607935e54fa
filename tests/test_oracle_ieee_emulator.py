"""Pins the oracle's per-operation arithmetic with an exact IEEE-754 emulator written
here from the standard, independent of numpy, of the C oracle and of the host FPU.

Every binary64 value is held as an exact ``Fraction``; each of the 6 (3-D) or 4 (2-D)
additions and the final multiplication of the update is computed EXACTLY and then
rounded to binary64 by ``rne`` below (round to nearest, ties to even: IEEE 754-2008
§4.3.1, integer mantissa arithmetic only -- no float operation produces a rounded
result).  The emulated iteration must equal ``oracle.jacobi3d`` / ``oracle.jacobi2d``
bit for bit.  This fixes, beyond any restatement of the formula in numpy:

* reading R3 -- the scale is ``x fl(1/7)`` (``x fl(1/5)`` in 2-D), not ``/ 7``;
* reading R4 -- the left-to-right order (c, x-, x+, y-, y+[, z-, z+]);
* reading R6 -- the fixed shell ("fixed borders").

The companion mutation checks run the emulator with the alternative readings and
assert that the oracle does NOT match them on the same data, so the pin would catch
an oracle that had drifted to any of them ("5-point average";
SURVEY.md §8(c.2) R2-R5)."""
from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

import jac_inputs as JI
import oracle

K7 = Fraction(0x12492492492492, 2 ** 55)   # 0x1.2492492492492p-3 = fl(1/7), from its bits
K5 = Fraction(0x1999999999999A, 2 ** 55)   # 0x1.999999999999ap-3 = fl(1/5)


def test_constants_are_the_hex_literals():
    assert K7 == Fraction(float.fromhex("0x1.2492492492492p-3"))
    assert K5 == Fraction(float.fromhex("0x1.999999999999ap-3"))
    # and they are the round-to-nearest values of 1/7 and 1/5
    assert rne(Fraction(1, 7)) == K7 and rne(Fraction(1, 5)) == K5


def rne(x: Fraction) -> Fraction:
    """The binary64 value nearest to x, ties to even (normal and subnormal range;
    overflow is not reached by these fields).  Integer arithmetic only."""
    if x == 0:
        return Fraction(0)
    sign = -1 if x < 0 else 1
    a = abs(x)
    # exponent e with 2^52 <= a / 2^e < 2^53, clamped at the subnormal exponent -1074
    e = a.numerator.bit_length() - a.denominator.bit_length() - 53
    while a / Fraction(2) ** e >= 2 ** 53:
        e += 1
    while a / Fraction(2) ** e < 2 ** 52:
        e -= 1
    e = max(e, -1074)
    m = a / Fraction(2) ** e
    q, r = divmod(m.numerator, m.denominator)          # m = q + r / den
    twice = 2 * r
    if twice > m.denominator or (twice == m.denominator and q % 2 == 1):
        q += 1
    return sign * Fraction(q) * Fraction(2) ** e       # q == 2^53 is still exact


def to_fracs(u: np.ndarray):
    return [Fraction(float(v)) for v in u.ravel()]


def emulate3d(u0: np.ndarray, n: int, scale=K7, order=(0, 1, 2, 3, 4, 5, 6), exact_div=False):
    """n Jacobi sweeps of the padded field, one rounding per operation."""
    nz2, ny2, nx2 = u0.shape
    A = to_fracs(u0)
    sx, sxy = nx2, nx2 * ny2
    for _ in range(n):
        B = list(A)  # shell copied, never written
        for k in range(1, nz2 - 1):
            for j in range(1, ny2 - 1):
                for i in range(1, nx2 - 1):
                    p = k * sxy + j * sx + i
                    terms = [A[p], A[p - 1], A[p + 1], A[p - sx], A[p + sx], A[p - sxy], A[p + sxy]]
                    s = terms[order[0]]
                    for t in order[1:]:
                        s = rne(s + terms[t])
                    B[p] = rne(s / 7) if exact_div else rne(s * scale)
        A = B
    return np.array([float(v) for v in A]).reshape(u0.shape)   # exact: every value is binary64


def emulate2d(u0: np.ndarray, n: int, scale=K5, order=(0, 1, 2, 3, 4), exact_div=False):
    ny2, nx2 = u0.shape
    A = to_fracs(u0)
    for _ in range(n):
        B = list(A)
        for j in range(1, ny2 - 1):
            for i in range(1, nx2 - 1):
                p = j * nx2 + i
                terms = [A[p], A[p - 1], A[p + 1], A[p - nx2], A[p + nx2]]
                s = terms[order[0]]
                for t in order[1:]:
                    s = rne(s + terms[t])
                B[p] = rne(s / 5) if exact_div else rne(s * scale)
        A = B
    return np.array([float(v) for v in A]).reshape(u0.shape)


def same_bits(a, b):
    return np.array_equal(a.view(np.uint64), b.view(np.uint64))


# ------------------------------------------------------------------ the emulator itself
def test_rne_against_known_roundings():
    """rne on cases whose binary64 roundings are fixed by the standard: exact values,
    halfway cases in both directions, the smallest subnormal, 0.1."""
    one = Fraction(1)
    ulp1 = Fraction(1, 2 ** 52)
    assert rne(one) == one
    assert rne(one + ulp1 / 2) == one                    # tie -> even (1.0)
    assert rne(one + 3 * ulp1 / 2) == one + 2 * ulp1     # tie -> even (mantissa ...10)
    assert rne(one + ulp1 / 2 + Fraction(1, 2 ** 80)) == one + ulp1
    assert rne(Fraction(1, 10)) == Fraction(3602879701896397, 2 ** 55)  # 0x1.999999999999ap-4
    assert rne(Fraction(1, 2 ** 1074)) == Fraction(1, 2 ** 1074)
    assert rne(Fraction(1, 2 ** 1075)) == 0                              # tie -> even (0)
    assert rne(Fraction(3, 2 ** 1076)) == Fraction(1, 2 ** 1074)
    assert rne(-Fraction(1, 3)) == -rne(Fraction(1, 3))
    assert rne(Fraction(2 ** 53 + 1)) == Fraction(2 ** 53)               # tie -> even
    assert rne(Fraction(2 ** 53 + 3)) == Fraction(2 ** 53 + 4)


# ------------------------------------------------------------------ pins of the oracle
@pytest.mark.parametrize("dims,n,seed", [((6, 5, 4), 3, 1), ((3, 4, 5), 4, 2), ((1, 1, 1), 2, 3)])
def test_oracle3d_equals_ieee_emulator(dims, n, seed):
    u0 = JI.hash_field(*dims, seed=seed)
    assert same_bits(oracle.jacobi3d(u0, n), emulate3d(u0, n))


@pytest.mark.parametrize("dims,n,seed", [((6, 5), 4, 1), ((9, 2), 5, 2), ((1, 1), 3, 3)])
def test_oracle2d_equals_ieee_emulator(dims, n, seed):
    u0 = JI.hash_field2d(*dims, seed=seed)
    assert same_bits(oracle.jacobi2d(u0, n), emulate2d(u0, n))


def test_oracle3d_emulator_on_signed_values():
    """Mixed signs and magnitudes (cancellation, different exponents per operand)."""
    rng = np.random.default_rng(11)
    u0 = rng.standard_normal((6, 5, 7)) * np.exp2(rng.integers(-8, 9, (6, 5, 7)))
    assert same_bits(oracle.jacobi3d(u0, 3), emulate3d(u0, 3))


# ------------------------------------------------------------------ mutations are caught
def test_mutations_3d_are_distinguished():
    """Each plausible misreading yields different bits on the same 6x5x4 field, so the
    emulator pin above would fail for an oracle that used it."""
    u0 = JI.hash_field(6, 5, 4, seed=1)
    got = oracle.jacobi3d(u0, 3)
    assert not same_bits(got, emulate3d(u0, 3, exact_div=True))                  # "/ 7"
    assert not same_bits(got, emulate3d(u0, 3, order=(1, 2, 3, 4, 5, 6, 0)))     # centre last
    assert not same_bits(got, emulate3d(u0, 3, order=(0, 5, 6, 3, 4, 1, 2)))     # z, y, x order
    assert not same_bits(got, emulate3d(u0, 3, scale=Fraction(1, 7)))            # unrounded 1/7


def test_mutations_2d_are_distinguished():
    u0 = JI.hash_field2d(6, 5, seed=1)
    got = oracle.jacobi2d(u0, 4)
    assert not same_bits(got, emulate2d(u0, 4, exact_div=True))                  # "/ 5"
    assert not same_bits(got, emulate2d(u0, 4, order=(1, 2, 3, 4, 0)))           # centre last
    assert not same_bits(got, emulate2d(u0, 4, order=(0, 3, 4, 1, 2)))           # y before x
