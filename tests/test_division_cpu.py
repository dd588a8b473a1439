"""Pins of the table division (R9), on CPU.

The fp32 kernels divide the PML numerator n by a table value B_d (= fp32(1 +
eta_d dt)) as
    q0 = RN(n * rB),  e = RN(n - q0 * B) (one FMA),  q = RN(q0 + e * rB) (one FMA)
with rB = RN(1 / B) from the host table.  A20 admits this only if it is
bitwise the IEEE quotient RN(n / B).  Here, independently of the GPU:

* rB is the correctly rounded reciprocal (exact rational comparison);
* the three-step quotient, emulated EXACTLY (products of two fp32 values are
  exact in fp64; the residual is exact; the final sum is re-done with exact
  rationals wherever fp64 rounding could land on an fp32 midpoint), equals
  RN(n / B) computed with exact integer arithmetic -- for every B_d of the
  C1/C2/C3/SPEC48/RAGGED tables and a dense sample of significands (every
  64th of the 2^23, plus both ends of the binade) in the binades the device
  check also covers.
The device-side proof is exhaustive (k_divcheck over all 2^23 significands at
plan setup); this test pins the arithmetic claim itself.
"""
from fractions import Fraction

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def _desc(name):
    from paper_2009_04619_b200 import _abi
    s = synth.scenario(name)
    return _abi.make_desc(s.nx, s.ny, s.nz, s.w, s.h, float(np.float32(s.dt)), s.eta_max)


def _rn_div(n: np.ndarray, B: np.float32) -> np.ndarray:
    """RN-even(n / B) for positive normal fp32 n (and a normal result), exact
    integer arithmetic: n = N 2^a, B = M 2^b with 24-bit N, M."""
    N, a = np.frexp(n.astype(np.float64))          # n = N * 2^a, N in [0.5, 1)
    Nm = (N * 2.0 ** 24).astype(np.int64)           # 24-bit integer significand
    Mf, b = np.frexp(np.float64(B))
    M = int(Mf * 2 ** 24)
    # q = Nm * 2^(a-24) / (M * 2^(b-24)) = (Nm / M) * 2^(a-b); take 26 quotient bits
    sh = 26
    num = Nm << sh
    Q = num // M
    rem = num - Q * M
    # normalise Q to 24 bits with round-to-nearest-even, tracking the exponent
    out = np.empty(n.shape, np.float32)
    for i in range(n.size):                          # vector sizes here are modest
        q, r = int(Q.flat[i]), int(rem.flat[i])
        e = int(a.flat[i]) - int(b) - sh
        nb = q.bit_length()
        drop = nb - 24
        keep = q >> drop
        low = q & ((1 << drop) - 1)
        half = 1 << (drop - 1)
        if low > half or (low == half and (r > 0 or keep & 1)):
            keep += 1
        out.flat[i] = np.float32(np.ldexp(float(keep), e + drop))
    return out


def _markstein(n: np.ndarray, B: np.float32, rB: np.float32) -> np.ndarray:
    n64, B64, rB64 = n.astype(np.float64), np.float64(B), np.float64(rB)
    q0 = (n64 * rB64).astype(np.float32)             # exact product, one rounding
    e = (n64 - q0.astype(np.float64) * B64).astype(np.float32)   # exact residual, one rounding
    s = q0.astype(np.float64) + e.astype(np.float64) * rB64      # e*rB exact; the sum may round
    q = s.astype(np.float32)
    # fp64 rounding of the sum can only mislead the fp32 rounding if it lands
    # exactly on an fp32 midpoint: redo those with exact rationals
    lo = q.astype(np.float64)
    nxt = np.nextafter(q, np.float32(np.inf) * np.sign(q)).astype(np.float64)
    prv = np.nextafter(q, np.float32(0)).astype(np.float64)
    mid = (s == (lo + nxt) / 2) | (s == (lo + prv) / 2)
    for i in np.nonzero(mid.ravel())[0]:
        exact = Fraction(float(q0.flat[i])) + Fraction(float(e.flat[i])) * Fraction(float(rB))
        cands = [np.float32(x) for x in (float(prv.flat[i]), float(lo.flat[i]), float(nxt.flat[i]))]
        best = min(cands, key=lambda c: (abs(Fraction(float(c)) - exact),
                                         int(np.float32(c).view(np.uint32)) & 1))
        q.flat[i] = best
    return q


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "SPEC48", "RAGGED"])
def test_reciprocal_table_is_correctly_rounded(name):
    from paper_2009_04619_b200 import _abi
    B, rB = _abi.wave_division_table(_desc(name))
    assert B[0] == 1.0 and rB[0] == 1.0 and np.all(B >= 1.0)
    for b, r in zip(B, rB):
        exact = 1 / Fraction(float(b))
        err = abs(Fraction(float(r)) - exact)
        for nb in (np.nextafter(r, np.float32(0)), np.nextafter(r, np.float32(2))):
            assert err < abs(Fraction(float(nb)) - exact), (b, r)


@pytest.mark.parametrize("name", ["C3", "C2", "RAGGED"])
def test_markstein_quotient_equals_ieee_division(name):
    from paper_2009_04619_b200 import _abi
    B, rB = _abi.wave_division_table(_desc(name))
    m = np.concatenate([np.arange(0, 1 << 23, 64), np.arange((1 << 23) - 64, 1 << 23)]).astype(np.uint32)
    bad = 0
    for exp in (127, 47):                            # binades [1, 2) and [2^-80, 2^-79)
        n = ((np.uint32(exp) << np.uint32(23)) | m).view(np.float32)
        for b, r in zip(B[1:], rB[1:]):              # B_0 = 1 divides exactly
            sel = slice(None, None, 7) if exp == 47 else slice(None)
            nn = n[sel]
            got = _markstein(nn, b, r)
            ref = _rn_div(nn[:4096], b) if exp == 127 else _rn_div(nn[:512], b)
            bad += int(np.sum(got[:ref.size].view(np.uint32) != ref.view(np.uint32)))
            # the whole sample against the fp64 quotient rounded to fp32: n / B
            # is never an fp32 midpoint (B * midpoint has more than 24
            # significant bits), so this single rounding can differ from RN
            # only if n / B lies within 2^-53 (relative) of one
            q64 = (nn.astype(np.float64) / np.float64(b)).astype(np.float32)
            bad += int(np.sum(got.view(np.uint32) != q64.view(np.uint32)))
    assert bad == 0
