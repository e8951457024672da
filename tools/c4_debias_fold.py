"""Can the quantiser's debias FADD2 be folded into the decision constant?  (VERDICT r1, C4 item.)

The kernel decides k = RN(Y c') with t = fma(y, c', 1.5 2^23) on y = b - KF, b = 2^23 + 2^15 + Y the
magic-exponent float of a biased SWAR coefficient (R10, kernels compress_quant_resid).  A
folded form would feed b straight in: t' = fma(b, c', A) with A = RN(1.5 2^23 - KF c').  In exact
arithmetic b c' + A = Y c' + 1.5 2^23 + eps with eps = A - (1.5 2^23 - KF c'), |eps| <= 1/2 (A lies in
[2^23, 2^24), spacing 1), so the folded decision is RN(Y c' + eps): it moves every threshold by eps.
This script counts the positions / values where the folded decision differs from the kernel's exact
one over every reachable Y (the P14 domain) at q = 16, in 64-bit-mantissa arithmetic (each fma is
exact before its one rounding to fp32).

    python tools/c4_debias_fold.py [q]      -> profiles/r02_c4_debias_fold.txt
"""
import os
import sys
from fractions import Fraction

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
T = np.loadtxt(os.path.join(ROOT, "tests", "golden", "c0_matrix.txt"), dtype=np.int64)
D = [8, 6, 4, 6, 8, 6, 4, 6]  # row norms^2 of T
M = np.float32(12582912.0)    # 1.5 2^23
KF = np.float32(8421376.0)    # 2^23 + 2^15


def c_prime(q, dd):
    """Smallest fp32 strictly above 1 / (q sqrt dd) (R10), compared exactly: f > 1/(q sqrt dd) <=> (f q)^2 dd > 1."""
    f = np.float32(1.0 / (q * np.sqrt(dd)))
    while (Fraction(float(f)) * Fraction(q)) ** 2 * dd > 1:
        f = np.nextafter(f, np.float32(0))
    while not (Fraction(float(f)) * Fraction(q)) ** 2 * dd > 1:
        f = np.nextafter(f, np.float32(np.inf))
    return f


def rn32(x):
    return x.astype(np.float32)


def main():
    q = float(sys.argv[1]) if len(sys.argv) > 1 else 16.0
    L = np.longdouble
    tot = bad = 0
    worst = []
    for i in range(8):
        for j in range(8):
            P = np.outer(T[i], T[j])
            lo, hi = int(255 * P[P < 0].sum()), int(255 * P[P > 0].sum())
            Y = np.arange(lo, hi + 1, dtype=np.int64)
            cc = c_prime(q, D[i] * D[j])
            # kernel: y exact, one fma rounding
            k_ker = rn32(Y.astype(L) * L(cc) + L(M)).astype(np.float64) - float(M)
            # folded: b = KF + Y exact in fp32 (|Y| < 2^15), A = RN(M - KF c')
            A = np.float32(L(M) - L(KF) * L(cc))
            b = (L(KF) + Y.astype(L))
            # b c' + A = Y c' + 1.5 2^23 + eps: the folded t' - 1.5 2^23 is the decision RN(Y c' + eps)
            eps = float(L(A) - (L(M) - L(KF) * L(cc)))
            k_fold = rn32(b * L(cc) + L(A)).astype(np.float64) - float(M)
            n_bad = int((k_fold != k_ker).sum())
            tot += len(Y)
            bad += n_bad
            worst.append((n_bad, i, j, len(Y), eps))
    print(f"# q = {q}: folded decision fma(b, c', RN(1.5 2^23 - KF c')) vs the kernel's fma(Y, c', 1.5 2^23)")
    print(f"# reachable (position, Y) pairs: {tot}; decisions that differ: {bad} ({bad / tot:.1%})")
    print("# position | reachable Y | differing | eps = A - (1.5 2^23 - KF c') (threshold shift)")
    for n_bad, i, j, n, eps in sorted(worst, reverse=True)[:16]:
        print(f"({i},{j}) | {n} | {n_bad} | {eps:+.4f}")


if __name__ == "__main__":
    main()
