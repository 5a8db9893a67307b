#!/usr/bin/env python
"""Generate the 2^(k/128) table of csrc/libm_exact.cuh.

glibc's exp (sysdeps/ieee754/dbl-64/e_exp.c, the ARM optimized-routines algorithm,
glibc >= 2.28) scales exp(r) by 2^(k/N), N = 128, read from a table of pairs
  tab[2k]   = bits of T_k, the relative tail: 2^(k/N) = H_k (1 + T_k)
  tab[2k+1] = bits of H_k (2^(k/N) rounded to nearest) - (k << 52) / N
These are mathematical constants; this script derives them at 80 digits and prints
the C initialiser.  tests/test_refcdf.py checks the device exp built on them against
the host libm bit for bit.
"""
import struct
from decimal import Decimal, getcontext

getcontext().prec = 80
N = 128


def bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def table():
    out = []
    for k in range(N):
        v = Decimal(2) ** (Decimal(k) / Decimal(N))
        h = float(v)  # correctly rounded (CPython's decimal -> float)
        t = float((v - Decimal(h)) / Decimal(h))
        out.append((bits(t), (bits(h) - ((k << 52) // N)) & 0xFFFFFFFFFFFFFFFF))
    return out


if __name__ == "__main__":
    rows = table()
    for i in range(0, N, 2):
        print("    " + " ".join(f"0x{t:016x}ull, 0x{h:016x}ull," for t, h in rows[i:i + 2]))
