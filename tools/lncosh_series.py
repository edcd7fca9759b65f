"""The small-argument series of lncosh / tanh used by the CUDA kernels (csrc/common.cuh,
lncosh_series / tanh_series): derives the coefficients c_n = 2^{2n}(2^{2n}-1) B_{2n} / (2n (2n)!)
exactly from the Bernoulli numbers, checks the constants written in common.cuh against them,
and measures the truncated series (evaluated in float64 by Horner in w = z^2) against 40-digit
mpmath log(cosh z) and tanh z on |z| <= 1/4.   python tools/lncosh_series.py"""
import os
import re
from fractions import Fraction
from math import comb, factorial

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_TERMS = 11


def coefficients(n_terms=N_TERMS):
    B = [Fraction(0)] * (2 * n_terms + 2)
    B[0] = Fraction(1)
    for m in range(1, 2 * n_terms + 2):
        B[m] = -sum(comb(m + 1, k) * B[k] for k in range(m)) / Fraction(m + 1)
    c = [Fraction(2 ** (2 * n) * (2 ** (2 * n) - 1)) * B[2 * n] / Fraction(2 * n * factorial(2 * n))
         for n in range(1, n_terms + 1)]
    return c, [2 * (n + 1) * x for n, x in enumerate(c)]


def header_constants():
    src = open(os.path.join(ROOT, "paper_2510_08430_b200", "csrc", "common.cuh")).read()
    out = {}
    for name in ("c", "t"):
        m = re.search(r"const double %s\[11\] = \{([^}]*)\}" % name, src)
        out[name] = [float(x) for x in m.group(1).replace("\n", " ").split(",")]
    return out


def horner(coef, w):
    acc = np.full_like(w, coef[-1])
    for x in coef[-2::-1]:
        acc = acc * w + x
    return acc


def max_rel_errors(n=3000, seed=0):
    import mpmath
    mpmath.mp.dps = 40
    rng = np.random.default_rng(seed)
    z = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    z = z / np.abs(z) * 0.25 * np.sqrt(rng.uniform(0, 1, n))
    z[:20] *= 1e-4
    h = header_constants()
    w = z * z
    lc = horner(h["c"], w) * w
    th = horner(h["t"], w) * z
    ref_l = np.array([complex(mpmath.log(mpmath.cosh(mpmath.mpc(x.real, x.imag)))) for x in z])
    ref_t = np.array([complex(mpmath.tanh(mpmath.mpc(x.real, x.imag))) for x in z])
    return float(np.max(np.abs(lc - ref_l) / np.abs(ref_l))), float(np.max(np.abs(th - ref_t) / np.abs(ref_t)))


if __name__ == "__main__":
    c, t = coefficients()
    h = header_constants()
    print("constants match:", all(float(a) == b for a, b in zip(c, h["c"])) and all(float(a) == b for a, b in zip(t, h["t"])))
    print("max relative error on |z| <= 1/4 (lncosh, tanh): %.3g %.3g" % max_rel_errors())
