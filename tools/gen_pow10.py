#!/usr/bin/env python3
"""Cached powers of ten for the Grisu2 double formatter in host_container.cpp:
10^k for k = -300, -292, ..., 324 as a normalised 64-bit significand f
(rounded to nearest) and binary exponent e with 10^k ~= f * 2^e. Exact
rational arithmetic; prints the C++ initialiser rows."""
from fractions import Fraction


def table():
    out = []
    for k in range(-300, 325, 8):
        c = Fraction(10) ** k
        e = c.numerator.bit_length() - c.denominator.bit_length() - 64
        while c / Fraction(2) ** e >= 2 ** 64:
            e += 1
        while c / Fraction(2) ** e < 2 ** 63:
            e -= 1
        q = c / Fraction(2) ** e
        f = int(q) + (1 if q - int(q) >= Fraction(1, 2) else 0)
        out.append((f, e, k))
    return out


if __name__ == "__main__":
    for f, e, k in table():
        print("    {0x%016XULL, %d, %d}," % (f, e, k))
