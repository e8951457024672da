"""Instrumented host model of the 22-addition fast algorithm (test-only).

Fig. 1 of the paper is missing from the LaTeX source; DESIGN.md
reading R2 derives an 8 + 6 + 8 = 22-addition flow graph for C0 . x from the displayed
matrix.  This module writes that graph out with an addition counter so the pins can check
(a) it equals C0 . x on all unit vectors and random integer vectors, and (b) it uses
exactly the 22 additions of Table 1 — and likewise for the transposed graph
(C0^T . X) used by the inverse.  The CUDA kernels implement the same graph; the oracle does
not use it (the oracle multiplies matrices).
"""


class Counter:
    def __init__(self):
        self.adds = 0
        self.mults = 0
        self.shifts = 0

    def add(self, a, b):
        self.adds += 1
        return a + b

    def sub(self, a, b):
        self.adds += 1
        return a - b


def forward8(x, k: Counter):
    """X = C0 . x: stage 1 (8 adds), even part (6 adds), odd part (8 adds)."""
    a0, a1, a2, a3 = k.add(x[0], x[7]), k.add(x[1], x[6]), k.add(x[2], x[5]), k.add(x[3], x[4])
    b0, b1, b2, b3 = k.sub(x[0], x[7]), k.sub(x[1], x[6]), k.sub(x[2], x[5]), k.sub(x[3], x[4])
    s, t = k.add(a0, a3), k.add(a1, a2)
    X = [None] * 8
    X[0], X[4] = k.add(s, t), k.sub(s, t)
    X[2], X[6] = k.sub(a0, a3), k.sub(a2, a1)
    X[1] = k.add(k.add(b0, b1), b2)
    X[3] = k.sub(k.sub(b0, b2), b3)
    X[5] = k.add(k.sub(b0, b1), b3)
    X[7] = k.sub(k.sub(b2, b1), b3)
    return X


def inverse8(X, k: Counter):
    """x = C0^T . X (transposed graph): 2 + 4 + 8 + 8 = 22 adds."""
    p, q = k.add(X[0], X[4]), k.sub(X[0], X[4])
    a0, a3 = k.add(p, X[2]), k.sub(p, X[2])
    a1, a2 = k.sub(q, X[6]), k.add(q, X[6])
    b0 = k.add(k.add(X[1], X[3]), X[5])
    b1 = k.sub(k.sub(X[1], X[5]), X[7])
    b2 = k.add(k.sub(X[1], X[3]), X[7])
    b3 = k.sub(k.sub(X[5], X[3]), X[7])
    x = [None] * 8
    for n, (a, b) in enumerate(((a0, b0), (a1, b1), (a2, b2), (a3, b3))):
        x[n], x[7 - n] = k.add(a, b), k.sub(a, b)
    return x


def sdct_forward8(x, k: Counter):
    """X = sign(C) . x for the SDCT comparator (Table 1 P:288-289 "24 additions"): stage 1
    (8 adds), even rows (+ + + +, + + - -, + - - +, + - + -) on a as a 4-point Hadamard (8 adds),
    odd rows (+ + + +, + - - -, + - + +, + - + -) on b with shared b0 +- b1, b2 +- b3 (8 adds)."""
    a = [k.add(x[n], x[7 - n]) for n in range(4)]
    b = [k.sub(x[n], x[7 - n]) for n in range(4)]
    s01, d01, s23, d23 = k.add(a[0], a[1]), k.sub(a[0], a[1]), k.add(a[2], a[3]), k.sub(a[2], a[3])
    t, u, v, w = k.add(b[0], b[1]), k.sub(b[0], b[1]), k.add(b[2], b[3]), k.sub(b[2], b[3])
    X = [None] * 8
    X[0], X[2] = k.add(s01, s23), k.sub(s01, s23)
    X[4], X[6] = k.sub(d01, d23), k.add(d01, d23)
    X[1], X[3], X[5], X[7] = k.add(t, v), k.sub(u, v), k.add(u, v), k.add(u, w)
    return X


def sdct_inverse8(X, k: Counter):
    """x = sign(C)^T . X (transposed graph): 8 + 8 + 8 = 24 adds."""
    p, q, r, s = k.add(X[0], X[2]), k.sub(X[0], X[2]), k.add(X[4], X[6]), k.sub(X[4], X[6])
    a = [k.add(p, r), k.sub(p, r), k.sub(q, s), k.add(q, s)]
    g, h, i, j = k.add(X[1], X[3]), k.sub(X[1], X[3]), k.add(X[5], X[7]), k.sub(X[5], X[7])
    b = [k.add(g, i), k.sub(h, i), k.add(h, i), k.add(h, j)]
    x = [None] * 8
    for n in range(4):
        x[n], x[7 - n] = k.add(a[n], b[n]), k.sub(a[n], b[n])
    return x
