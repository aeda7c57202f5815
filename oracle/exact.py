"""Exact-rational (``fractions.Fraction``) statement of one D3Q19 LBGK pull step.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Pure-Python loops, for
boxes of a few cells.  It follows the same passages as ``lbm_oracle.c``:
P:407-425 (eq:lbm, eq:feq), P:443-448 (moments, u = j / rho0)
(centred PDFs), P:466-480 (pull, two grids), P:482-490 (half-way BB with the
delivered-direction reading R3 of DESIGN.md).  Its result is exact, so the
fp64 C oracle must match it to rounding (brute force on tiny inputs).
"""
from __future__ import annotations

from fractions import Fraction as Fr

# Frozen D3Q19 direction order (R2; checked against tests/golden/d3q19_table.txt).
E = [(0, 0, 0),
     (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1),
     (1, 1, 0), (-1, -1, 0), (1, -1, 0), (-1, 1, 0),
     (1, 0, 1), (-1, 0, -1), (1, 0, -1), (-1, 0, 1),
     (0, 1, 1), (0, -1, -1), (0, 1, -1), (0, -1, 1)]
W = [Fr(1, 3)] + [Fr(1, 18)] * 6 + [Fr(1, 36)] * 12
OPP = [0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17]
RHO0 = Fr(1)


def feq(drho, u):
    usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2]
    out = []
    for i in range(19):
        eu = E[i][0] * u[0] + E[i][1] * u[1] + E[i][2] * u[2]
        out.append(W[i] * (drho + RHO0 * (3 * eu + Fr(9, 2) * eu * eu - Fr(3, 2) * usq)))
    return out


def step(f, flags, wall_u, omega, periodic=(0, 0, 0)):
    """One step.  f: dict (x,y,z) -> list of 19 Fractions for interior cells;
    flags: dict (x,y,z) -> int for interior + shell cells (shell = -1..n);
    wall_u: list of 3-tuples of Fractions; omega: Fraction.  Returns new dict."""
    xs = sorted({c[0] for c in f})
    ys = sorted({c[1] for c in f})
    zs = sorted({c[2] for c in f})
    n = (len(xs), len(ys), len(zs))
    out = {}
    for c, fc in f.items():
        if flags[c] != 0:
            out[c] = list(fc)
            continue
        p = []
        for i in range(19):
            s = [c[a] - E[i][a] for a in range(3)]
            for a in range(3):
                if periodic[a]:
                    s[a] %= n[a]
            s = tuple(s)
            nb = flags[s]
            if nb == 0:
                p.append(f[s][i])
            elif nb == 1:
                p.append(fc[OPP[i]])
            else:
                uw = wall_u[nb - 2]
                eu = E[i][0] * uw[0] + E[i][1] * uw[1] + E[i][2] * uw[2]
                p.append(fc[OPP[i]] + 6 * W[i] * RHO0 * eu)
        drho = sum(p, Fr(0))
        u = [sum((E[i][a] * p[i] for i in range(19)), Fr(0)) / RHO0 for a in range(3)]
        fe = feq(drho, u)
        out[c] = [p[i] - omega * (p[i] - fe[i]) for i in range(19)]
    return out
