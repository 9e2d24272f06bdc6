"""Coefficients of the table-free erfcx used by the fused short-range kernel.

    erfcx(x) = P(u),  t = (x - K) / (x + K),  u = (t - tm) / th  in [-1, 1]

for x in [0, XMAX] (t in [-1, t_max]), P a degree-DEG polynomial interpolating at
Chebyshev nodes (50-digit mpmath), evaluated by Horner in double.  The rational
map flattens erfcx's decay so one polynomial covers the whole range (degree 19
for 2e-16 on [0, 6] with K = 4), with UNIFORM coefficients: no per-lane table
reads (a shared-memory coefficient load costs >= 2 wavefronts per warp, which
made the table forms shared-memory bound in the pair kernel).

    python tools/gen_erfcx_rational.py [DEG] [K] [XMAX]  -> prints a C array + the error
"""

import sys

import mpmath as mp
import numpy as np

mp.mp.dps = 50
DEG = int(sys.argv[1]) if len(sys.argv) > 1 else 19
K = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
XMAX = float(sys.argv[3]) if len(sys.argv) > 3 else 6.0


def erfcx(x):
    x = mp.mpf(x)
    return mp.exp(x * x) * mp.erfc(x)


def main():
    t0, t1 = mp.mpf(-1), (mp.mpf(XMAX) - K) / (mp.mpf(XMAX) + K)
    tm, th = (t0 + t1) / 2, (t1 - t0) / 2
    nodes = [mp.cos(mp.pi * (mp.mpf(j) + mp.mpf(1) / 2) / (DEG + 1)) for j in range(DEG + 1)]
    xs = []
    for u in nodes:
        t = tm + th * u
        xs.append(K * (1 + t) / (1 - t))
    V = mp.matrix([[u ** j for j in range(DEG + 1)] for u in nodes])
    c = mp.lu_solve(V, mp.matrix([erfcx(x) for x in xs]))
    coef = [float(c[j]) for j in range(DEG + 1)]
    worst = 0.0
    for x in np.linspace(0.0, XMAX, 4001):
        t = (x - K) / (x + K)
        u = (t - float(tm)) / float(th)
        p = 0.0
        for cj in reversed(coef):
            p = p * u + cj
        worst = max(worst, abs(float((mp.mpf(p) - erfcx(x)) / erfcx(x))))
    print(f"// degree {DEG}, K = {K}, x in [0, {XMAX}]: max rel err {worst:.3g}")
    print(f"// t = (x - K)/(x + K), u = (t - ({float(tm)!r})) / {float(th)!r}")
    print("{" + ", ".join(f"{v:.17e}" for v in coef) + "}")


if __name__ == "__main__":
    main()
