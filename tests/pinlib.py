"""Shared helpers for the oracle pins (no oracle arithmetic here)."""
import json
import math
import os
import struct
from fractions import Fraction

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def f32(v):
    return struct.unpack("f", struct.pack("f", v))[0]


def ulp32(v):
    v = abs(f32(v))
    if v == 0:
        return 2.0 ** -149
    e = math.frexp(v)[1] - 1
    return 2.0 ** (e - 23)


def dempster_by_sets(a, b):
    """Dempster's rule from its set-theoretic definition (Dempster 1968; Eq. 63 cites it):
    m(C) = sum_{A cap B = C} m1(A) m2(B) / (1 - sum_{A cap B = {}} m1(A) m2(B)), on the frame
    {O, F} with focal sets {O}, {F}, {O,F}.  Exact rational arithmetic."""
    O, F = frozenset("O"), frozenset("F")
    Om = O | F
    m1 = {O: Fraction(a[0]), F: Fraction(a[1]), Om: 1 - Fraction(a[0]) - Fraction(a[1])}
    m2 = {O: Fraction(b[0]), F: Fraction(b[1]), Om: 1 - Fraction(b[0]) - Fraction(b[1])}
    out = {O: Fraction(0), F: Fraction(0), Om: Fraction(0)}
    conflict = Fraction(0)
    for A, x in m1.items():
        for B, y in m2.items():
            Cs = A & B
            if Cs:
                out[Cs] += x * y
            else:
                conflict += x * y
    return float(out[O] / (1 - conflict)), float(out[F] / (1 - conflict))


