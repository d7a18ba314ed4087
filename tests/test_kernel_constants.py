"""CPU checks of constant tables written into the CUDA sources (no GPU, no oracle):
the Bernoulli-series coefficients of the Planck integral in k_trt.cu are compared with
exact Bernoulli numbers (rational arithmetic), and the series/tail switch is checked
to keep both branches inside their accuracy range."""
from __future__ import annotations

import math
import os
import re
from fractions import Fraction
from math import comb, factorial

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2504_21784_b200", "csrc", "k_trt.cu")


def bernoulli(n: int) -> list[Fraction]:
    B = [Fraction(0)] * (n + 1)
    B[0] = Fraction(1)
    for m in range(1, n + 1):
        B[m] = -sum(comb(m + 1, k) * B[k] for k in range(m)) / Fraction(m + 1)
    return B


def table():
    src = open(SRC).read()
    body = re.search(r"constexpr double c\[(\d+)\] = \{(.*?)\};", src, re.S)
    assert body, "coefficient table not found in k_trt.cu"
    vals = [v.strip() for v in body.group(2).replace("\n", " ").split(",") if v.strip()]
    out = []
    for v in vals:
        v = re.sub(r"//.*", "", v).strip()
        out.append(1.0 / 3.0 if v == "1.0 / 3.0" else float.fromhex(v))
    return int(body.group(1)), out


def test_bernoulli_table_exact():
    n, c = table()
    assert n == len(c) == 26
    B = bernoulli(2 * (n - 1))
    assert c[0] == 1.0 / 3.0
    for j in range(1, n):
        exact = B[2 * j] / (factorial(2 * j) * (2 * j + 3))
        assert c[j] == float(exact), j            # correctly rounded once


def planck_series(x: float, c) -> float:
    # the kernel's x < switch branch, in Python double arithmetic
    x2 = x * x
    s = c[-1]
    for j in range(len(c) - 2, 0, -1):
        s = s * x2 + c[j]
    return 15 / math.pi ** 4 * x ** 3 * (c[0] - x * 0.125 + s * x2)


def planck_tail(x: float, full: bool = False) -> float:
    # the kernel's x >= switch branch (full: 80 terms, the reference for both branches)
    t = 0.0
    en, e1 = 1.0, math.exp(-x)
    for n in range(1, (80 if full else min(14, int(38.0 / x) + 2)) + 1):
        rn = 1.0 / n
        en *= e1
        t += en * rn * (rn * (rn * (6 * rn + 6 * x) + 3 * x * x) + x ** 3)
    return 1.0 - 15 / math.pi ** 4 * t


def test_series_and_tail_agree_at_the_switch():
    """Both expansions of P(x) = 15/pi^4 int_0^x t^3/(e^t - 1) dt (PAPER.md eq:planck) at
    the switch x = 3 and around it: two independent series must agree to rounding."""
    _, c = table()
    src = open(SRC).read()
    assert "if (x < 3.0)" in src
    for x in (1.0, 2.0, 2.5, 2.9, 2.999):
        a, b = planck_series(x, c), planck_tail(x, full=True)
        assert abs(a - b) <= 4e-15 * b, (x, a, b)
    for x in (3.0, 3.5, 5.0, 12.0, 40.0):
        a, b = planck_tail(x), planck_tail(x, full=True)
        assert abs(a - b) <= 1e-16 * b, (x, a, b)


def test_planck_limits():
    _, c = table()
    # small x: P ~ (15/pi^4) x^3 / 3; large x: P -> 1 (Stefan-Boltzmann normalisation)
    x = 1e-3
    assert abs(planck_series(x, c) / (15 / math.pi ** 4 * x ** 3 / 3) - 1) < 1e-3
    assert abs(planck_tail(60.0) - 1.0) < 1e-15
