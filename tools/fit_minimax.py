"""Near-minimax coefficients of the fast exp / sincos polynomials (fastmath.cuh,
SLAB_MINIMAX): Chebyshev fits in mpmath on the reduced ranges, then the max
relative error of the double-precision Horner evaluation (correctly rounded
FMAs) against mpmath on a dense grid.

    python tools/fit_minimax.py

e^r = 1 + r (1 + r E(r)), |r| <= ln2/2, E degree 9;
sin r = r + r z P(z), cos r = 1 + z Q(z), z = r^2, |r| <= pi/4, P degree 5, Q degree 6.
"""
import mpmath as mp
import numpy as np

mp.mp.dps = 50


def fit(f, a, b, deg):
    c = mp.chebyfit(f, [a, b], deg + 1)
    return [float(x) for x in c]  # highest degree first


def fma(a, b, c):  # correctly rounded
    return float(mp.mpf(a) * mp.mpf(b) + mp.mpf(c))


def horner(c, x):
    p = c[0]
    for k in c[1:]:
        p = fma(p, x, k)
    return p


def main():
    h, q = mp.log(2) / 2, mp.pi / 4
    E = fit(lambda r: (mp.exp(r) - 1 - r) / r**2 if r != 0 else mp.mpf(1) / 2, -h, h, 9)
    P = fit(lambda z: (mp.sin(mp.sqrt(z)) - mp.sqrt(z)) / mp.sqrt(z) ** 3 if z != 0
            else -mp.mpf(1) / 6, mp.mpf(0), q**2, 5)
    Q = fit(lambda z: (mp.cos(mp.sqrt(z)) - 1) / z if z != 0 else -mp.mpf(1) / 2,
            mp.mpf(0), q**2, 6)
    print("exp E:", E)
    print("sin P:", P)
    print("cos Q:", Q)
    ee = max(abs((fma(fma(horner(E, r), r, 1.0), r, 1.0) - mp.exp(r)) / mp.exp(r))
             for r in np.linspace(-float(h), float(h), 2001))
    es = ec = 0
    for r in np.linspace(-float(q), float(q), 2001):
        z = float(mp.mpf(r) * r)
        s = fma(horner(P, z) * z, r, r)
        c = fma(horner(Q, z), z, 1.0)
        if r != 0:
            es = max(es, abs((s - mp.sin(r)) / mp.sin(r)))
        ec = max(ec, abs((c - mp.cos(r)) / mp.cos(r)))
    print(f"max rel error: exp {float(ee):.3g}  sin {float(es):.3g}  cos {float(ec):.3g}")


if __name__ == "__main__":
    main()
