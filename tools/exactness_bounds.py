"""Exactness proof for the fp32 inverse of the fused compress kernel (R13/R17).

The kernel's zonal inverse runs the transposed 22-addition graph (columns, then rows) in fp32 on
integer-valued inputs V = W (.) Y (+ a DC bias).  Every node is then an integer, and fp32 is exact
as long as every node's magnitude stays below 2^24.  Each node is an affine function of the 64
pixels of a block, so its exact range over all uint8 blocks is [c + 255 sum(a-), c + 255 sum(a+)].
This script propagates those affine forms through the same graph, in the same operation order as
adct_device.cuh inv8 / inverse2d, for every r and both kernel variants:

  direct    V = W (.) M_r (.) Y, optionally plus 589824 on V_00 (so every output is R + 589824,
            and the f16 error route is one FMA: e = (R + 589824) - 576 (1024 + x) = R - 576 x),
            or plus 589824 + 1.5 2^23 (the exact-SSE kernel: R - 576 x + 1.5 2^23 in [2^23, 2^24))
  residual  V = W (.) (1 - M_r) (.) Y (the discarded coefficients): output = 576 x - R directly
            (576 x = C0^T (W (.) Y) C0 for every block, the r = 64 case of P8)

Prints the largest |node| per r and variant and exits non-zero if any reaches 2^24.
Pure host arithmetic on T (the displayed C0); it models the kernel, not the oracle.
"""
from __future__ import annotations

import sys

import numpy as np

T = np.array([[1, 1, 1, 1, 1, 1, 1, 1],
              [1, 1, 1, 0, 0, -1, -1, -1],
              [1, 0, 0, -1, -1, 0, 0, 1],
              [1, 0, -1, -1, 1, 1, 0, -1],
              [1, -1, -1, 1, 1, -1, -1, 1],
              [1, -1, 0, 1, -1, 0, 1, -1],
              [0, -1, 1, 0, 0, 1, -1, 0],
              [0, -1, 1, -1, 1, -1, 1, 0]], dtype=np.int64)
D = np.array([8, 6, 4, 6, 8, 6, 4, 6])
W = 576 // np.outer(D, D)
DC_BIASES = (0, 589824, 13172736)  # none, 576 * 1024 (the f16 error route of compress_inv), and
# 576 * 1024 + 1.5 * 2^23 (k_compress_exact: the error as the bit pattern of one float in [2^23, 2^24))


def zz(i: int, j: int) -> int:
    s = i + j
    before = sum((t + 1) if t < 8 else 15 - t for t in range(s))
    lo, hi = (0, s) if s < 8 else (s - 7, 7)
    return before + ((i - lo) if s & 1 else (hi - i))


class Bound:
    def __init__(self):
        self.max = 0

    def see(self, f):
        if f is None:
            return f
        a, c = f[:64], f[64]
        lo = c + 255 * a[a < 0].sum()
        hi = c + 255 * a[a > 0].sum()
        self.max = max(self.max, abs(lo), abs(hi))
        return f


def add(B, a, b):
    if a is None:
        return b
    if b is None:
        return a
    return B.see(a + b)


def sub(B, a, b):
    if b is None:
        return a
    if a is None:
        return -b
    return B.see(a - b)


def inv8(B, x):
    p, q = add(B, x[0], x[4]), sub(B, x[0], x[4])
    a0, a3 = add(B, p, x[2]), sub(B, p, x[2])
    a1, a2 = sub(B, q, x[6]), add(B, q, x[6])
    b0 = add(B, add(B, x[1], x[3]), x[5])
    b1 = sub(B, sub(B, x[1], x[5]), x[7])
    b2 = add(B, sub(B, x[1], x[3]), x[7])
    b3 = sub(B, sub(B, x[5], x[3]), x[7])
    return [add(B, a0, b0), add(B, a1, b1), add(B, a2, b2), add(B, a3, b3),
            sub(B, a3, b3), sub(B, a2, b2), sub(B, a1, b1), sub(B, a0, b0)]


def inv8s(B, x):
    """The one-instruction-butterfly graph (adct_device.cuh inv8s): the same outputs through the
    intermediate nodes x1 +- x3 and x5 +- x7 instead of inv8's (x1 + x3), (x1 - x5), (x1 - x3), (x5 - x3)."""
    p, q = add(B, x[0], x[4]), sub(B, x[0], x[4])
    a0, a3 = add(B, p, x[2]), sub(B, p, x[2])
    a2, a1 = add(B, q, x[6]), sub(B, q, x[6])
    s13p, s13m = add(B, x[1], x[3]), sub(B, x[1], x[3])
    s57p, s57m = add(B, x[5], x[7]), sub(B, x[5], x[7])
    b0, b1 = add(B, s13p, x[5]), sub(B, x[1], s57p)
    b2, b3 = add(B, s13m, x[7]), sub(B, s57m, x[3])
    return [add(B, a0, b0), add(B, a1, b1), add(B, a2, b2), add(B, a3, b3),
            sub(B, a3, b3), sub(B, a2, b2), sub(B, a1, b1), sub(B, a0, b0)]


GRAPHS = {"f32x2": (inv8, inv8), "scalar": (inv8s, inv8s), "hybrid": (inv8, inv8s)}  # (columns, rows)


def forms_Y():
    """Y_kl = sum_ij T_ki T_lj x_ij as affine forms (64 coefficients + constant)."""
    Y = np.zeros((8, 8, 65), dtype=np.int64)
    for k in range(8):
        for l in range(8):
            Y[k, l, :64] = np.outer(T[k], T[l]).reshape(64)
    return Y


def run(r: int, variant: str, bias: int = 0, graph: str = "f32x2"):
    B = Bound()
    Y = forms_Y()
    V = [[None] * 8 for _ in range(8)]
    for k in range(8):
        for l in range(8):
            kept = zz(k, l) < r
            live = kept if variant == "direct" else not kept
            if live:
                V[k][l] = B.see(W[k, l] * Y[k, l])
    if variant == "direct" and bias:
        V[0][0] = V[0][0].copy()
        V[0][0][64] += bias
        B.see(V[0][0])
    col, row = GRAPHS[graph]
    U = [col(B, [V[k][l] for k in range(8)]) for l in range(8)]
    out = [row(B, [U[l][i] for l in range(8)]) for i in range(8)]
    # check the final identity: direct -> R + bias, residual -> 576 x - R
    return B.max, out


def run_band_chain(row_graph=None):
    """k_compress_sweep_inc: e = 576 x, then for each anti-diagonal band b = 0..7 (r = 1, 3, ..., 36)
    e -= C0^T (W . [band b] . Y) C0 with the band's column inverse as a sign pattern (one coefficient
    per column) and its row inverse through inv8.  Returns (max |node|, final error forms per r)."""
    B = Bound()
    Y = forms_Y()
    e = []
    for i in range(8):
        row = []
        for n in range(8):
            f = np.zeros(65, dtype=np.int64)
            f[i * 8 + n] = 576
            row.append(f)
        e.append(row)
    finals = {}
    for band in range(8):
        for i in range(8):
            u = []
            for l in range(8):
                k = band - l
                if 0 <= k <= 7 and T[k, i] != 0:
                    u.append(B.see(T[k, i] * W[k, l] * Y[k, l]))
                else:
                    u.append(None)
            out = (row_graph or inv8)(B, u)
            e[i] = [sub(B, e[i][n], out[n]) for n in range(8)]
        finals[(band + 1) * (band + 2) // 2] = [row[:] for row in e]
    return B.max, finals


def main():
    worst = 0
    for graph in GRAPHS:  # the kernels' three inverse flavours (sinv_mode)
        for variant, bias in (("direct", 0), ("direct", DC_BIASES[1]), ("direct", DC_BIASES[2]), ("residual", 0)):
            row = []
            for r in range(1, 65):
                if variant == "residual" and r == 64:
                    continue
                m, _ = run(r, variant, bias, graph)
                worst = max(worst, m)
                row.append(f"{r}:{m}")
            print(graph, variant, f"bias={bias}", " ".join(row))
    for name, g in (("inv8", inv8), ("inv8s", inv8s)):
        m, _ = run_band_chain(g)
        worst = max(worst, m)
        print(f"band chain (k_compress_sweep_inc, row graph {name})", m)
    print("max |node| =", worst, "< 2^24 =", 1 << 24, "->", "EXACT" if worst < (1 << 24) else "NOT EXACT")
    return 0 if worst < (1 << 24) else 1


if __name__ == "__main__":
    sys.exit(main())
