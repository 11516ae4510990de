"""CPU restatement of the reference's generation noise (TEST INFRASTRUCTURE ONLY).

flowpipe draws each generation's initial latent with
``np.random.default_rng([seed, gen_id]).standard_normal(dim)`` (src/pipeline.py:92-98).
The algorithm lives in numpy (a dependency, ``numpy>=1.24`` unpinned in
pkg/pyproject.toml:10-12; numpy 2.3 here), not in the reference tree, so this
module restates numpy's published algorithm in exact Python integer / IEEE double
arithmetic and is pinned against numpy itself (tests/test_noise_oracle.py):

* SeedSequence (numpy/random/bit_generator.pyx): entropy ints -> little-endian
  uint32 words, ``mix_entropy`` into a 4-word pool with the hashmix / mix
  constants, ``generate_state(4, uint64)``.
* PCG64 (numpy/random/src/pcg64/pcg64.h): 128-bit LCG (multiplier
  0x2360ed051fc65da44385df649fccf645), ``srandom(initstate, initseq)``, XSL-RR
  64-bit output, step-then-output.
* ``random_standard_normal`` (numpy/random/src/distributions/distributions.c):
  256-level ziggurat with numpy's ki/wi/fi tables, the idx==0 tail via
  ``log1p`` and the wedge test via ``exp``.

``log1p`` here is the platform libm's (math.log1p == npy_log1p); the device kernel
carries its own restatement of this glibc's log1p, checked bit-for-bit against
math.log1p by tests/test_noise_oracle.py.

Only tests/, __graft_entry__.smoke() and tools/ may import this module.
"""

from __future__ import annotations

import math
import os
import re
import struct
from fractions import Fraction

import numpy as np

M128 = (1 << 128) - 1
M32 = 0xFFFFFFFF
PCG_MULT = (2549297995355413924 << 64) + 4865540595714422341

# SeedSequence constants (bit_generator.pyx)
INIT_A, MULT_A = 0x43B0D7E5, 0x931E8875
INIT_B, MULT_B = 0x8B51F9DD, 0x58F38DED
MIX_MULT_L, MIX_MULT_R = 0xCA01F9DD, 0x4973F715
XSHIFT = 16

ZIG_R = 3.6541528853610088
ZIG_INV_R = 0.27366123732975828

_HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_2511_22009_b200", "csrc", "ziggurat_tables.h")


def load_tables(path: str = _HDR):
    """(ki, wi, fi) parsed from the generated header (single source of the constants)."""
    txt = open(path).read()

    def block(name):
        body = re.search(name + r"\[256\] = \{(.*?)\};", txt, re.S).group(1)
        return [t.strip() for t in body.split(",") if t.strip()]

    ki = [int(v.rstrip("ULL"), 16) for v in block("SF_ZIG_KI")]
    wi = [float.fromhex(v) for v in block("SF_ZIG_WI")]
    fi = [float.fromhex(v) for v in block("SF_ZIG_FI")]
    return ki, wi, fi


def entropy_words(values) -> list[int]:
    """_coerce_to_uint32_array of a list of non-negative ints."""
    out = []
    for n in values:
        n = int(n)
        if n < 0:
            raise ValueError("expected non-negative integer")
        if n == 0:
            out.append(0)
        while n > 0:
            out.append(n & M32)
            n >>= 32
    return out


def seed_sequence_state(values, n_words64: int = 2 * 2) -> list[int]:
    """SeedSequence(values).generate_state(n_words64, np.uint64)."""
    ent = entropy_words(values)
    pool = [0, 0, 0, 0]
    hc = INIT_A

    def hashmix(v):
        nonlocal hc
        v = (v ^ hc) & M32
        hc = (hc * MULT_A) & M32
        v = (v * hc) & M32
        return v ^ (v >> XSHIFT)

    def mix(x, y):
        r = (MIX_MULT_L * x - MIX_MULT_R * y) & M32
        return r ^ (r >> XSHIFT)

    for i in range(4):
        pool[i] = hashmix(ent[i] if i < len(ent) else 0)
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    hb = INIT_B
    words = []
    for i in range(2 * n_words64):
        v = pool[i % 4]
        v = (v ^ hb) & M32
        hb = (hb * MULT_B) & M32
        v = (v * hb) & M32
        words.append(v ^ (v >> XSHIFT))
    return [words[2 * i] | (words[2 * i + 1] << 32) for i in range(n_words64)]


class PCG64:
    """numpy's PCG64 (XSL-RR 128/64) seeded from SeedSequence(values)."""

    def __init__(self, values):
        s = seed_sequence_state(values, 4)
        initstate = (s[0] << 64) | s[1]
        initseq = (s[2] << 64) | s[3]
        self.inc = ((initseq << 1) | 1) & M128
        self.state = 0
        self._step()
        self.state = (self.state + initstate) & M128
        self._step()

    def _step(self):
        self.state = (self.state * PCG_MULT + self.inc) & M128

    def next64(self) -> int:
        self._step()
        hi, lo = self.state >> 64, self.state & ((1 << 64) - 1)
        rot = self.state >> 122
        v = hi ^ lo
        return ((v >> rot) | (v << ((64 - rot) & 63))) & ((1 << 64) - 1)

    def next_double(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)


def standard_normal(rng: PCG64, n: int, tables=None) -> np.ndarray:
    ki, wi, fi = tables or load_tables()
    out = np.empty(n, dtype=np.float64)
    for i in range(n):
        while True:
            r = rng.next64()
            idx = r & 0xFF
            r >>= 8
            sign = r & 1
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = rabs * wi[idx]
            if sign:
                x = -x
            if rabs < ki[idx]:
                break
            if idx == 0:
                while True:
                    xx = -ZIG_INV_R * math.log1p(-rng.next_double())
                    yy = -math.log1p(-rng.next_double())
                    if yy + yy > xx * xx:
                        x = -(ZIG_R + xx) if (rabs >> 8) & 1 else ZIG_R + xx
                        break
                break
            if (fi[idx - 1] - fi[idx]) * rng.next_double() + fi[idx] < math.exp(-0.5 * x * x):
                break
        out[i] = x
    return out


def generation_noise(seed: int, gen_id: int, dim: int, tables=None) -> np.ndarray:
    """default_rng([seed, gen_id]).standard_normal(dim), restated."""
    return standard_normal(PCG64([seed, gen_id]), dim, tables)


# ---------------------------------------------------------------- glibc log1p restatement
# The device kernel (csrc/numpy_noise.cu glibc_log1p) restates the log1p of this
# platform's libm (glibc 2.39, x86-64 FMA ifunc variant, fdlibm-derived) operation for
# operation, from its disassembly; this is the same restatement in exact Python
# (fma via rationals), pinned bit-for-bit against math.log1p in tests/test_noise_oracle.py.

def _fma(a: float, b: float, c: float) -> float:
    r = Fraction(a) * Fraction(b) + Fraction(c)
    if r == 0:
        return a * b + c
    return r.numerator / r.denominator


def _hi(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", x))[0] >> 32


def _with_hi(x: float, hi: int) -> float:
    lo = struct.unpack("<Q", struct.pack("<d", x))[0] & 0xFFFFFFFF
    return struct.unpack("<d", struct.pack("<Q", ((hi & 0xFFFFFFFF) << 32) | lo))[0]


_LN2_HI, _LN2_LO = 6.93147180369123816490e-01, 1.90821492927058770002e-10
_LP = (6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01, 2.222219843214978396e-01,
       1.818357216161805012e-01, 1.531383769920937332e-01, 1.479819860511658591e-01)


def glibc_log1p(x: float) -> float:
    hx = _hi(x)
    if hx <= 0x3FDA8279:
        ax = hx & 0x7FFFFFFF
        if ax > 0x3FEFFFFF:
            return -math.inf if x == -1.0 else math.nan
        if ax <= 0x3E1FFFFF:
            return x if ax <= 0x3C8FFFFF else _fma(-(x * x), 0.5, x)
        if ((hx + 0x402D413C) & 0xFFFFFFFF) > 0x402D413C:
            return _log1p_poly(x, 0, 0.0)
    elif hx > 0x7FEFFFFF:
        return x + x
    u = x + 1.0
    h = _hi(u) & 0xFFFFFFFF
    k = (h >> 20) - 1023
    c = (1.0 - (u - x)) / u if k > 0 else (x - (u - 1.0)) / u
    hu = h & 0xFFFFF
    if hu <= 0x6A09D:
        u = _with_hi(u, hu | 0x3FF00000)
    else:
        k += 1
        u = _with_hi(u, hu | 0x3FE00000)
        hu = (0x100000 - hu) >> 2
    f = u - 1.0
    if hu != 0:
        return _log1p_poly(f, k, c)
    hfsq = (f * 0.5) * f
    kd = float(k)
    if f == 0.0:
        return 0.0 if k == 0 else _fma(kd, _LN2_HI, _fma(kd, _LN2_LO, c))
    R = _fma(-f, 0.6666666666666666, 1.0) * hfsq
    if k == 0:
        return f - R
    return _fma(kd, _LN2_HI, -((R - _fma(kd, _LN2_LO, c)) - f))


def _log1p_poly(f: float, k: int, c: float) -> float:
    lp1, lp2, lp3, lp4, lp5, lp6, lp7 = _LP
    hfsq = (f * 0.5) * f
    s = f / (f + 2.0)
    z = s * s
    R2, R3, R4 = _fma(z, lp3, lp2), _fma(z, lp5, lp4), _fma(z, lp7, lp6)
    z2 = z * z
    z4 = z2 * z2
    z6 = z2 * z4
    R = _fma(z6, R4, _fma(z4, R3, _fma(z, lp1, z2 * R2)))
    w = (R + hfsq) * s
    if k == 0:
        return f - (hfsq - w)
    kd = float(k)
    return _fma(kd, _LN2_HI, -((hfsq - (_fma(kd, _LN2_LO, c) + w)) - f))
