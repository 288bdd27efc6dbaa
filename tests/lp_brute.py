"""Brute-force vertex enumeration for tiny box LPs (test-only; independent of both
the oracle and the CUDA path).

min c^T x  s.t.  A x = b,  l <= x <= u. A basic solution picks m
linearly independent columns B, puts every nonbasic column at a finite bound and
solves A_B x_B = b - A_N x_N; it is a vertex iff l_B <= x_B <= u_B.
"""
import itertools

import numpy as np


def vertices(A, b, l, u, tol=1e-9):
    m, n = A.shape
    out = []
    for B in itertools.combinations(range(n), m):
        AB = A[:, B]
        if abs(np.linalg.det(AB)) < 1e-10:
            continue
        N = [j for j in range(n) if j not in B]
        choices = [[v for v in (l[j], u[j]) if np.isfinite(v)] for j in N]
        for assign in itertools.product(*choices):
            x = np.zeros(n)
            x[N] = assign
            rhs = b - A[:, N] @ np.array(assign) if N else b.copy()
            xB = np.linalg.solve(AB, rhs)
            if np.all(xB >= l[list(B)] - tol) and np.all(xB <= u[list(B)] + tol):
                x[list(B)] = xB
                out.append(x)
    uniq = []
    for x in out:
        if not any(np.allclose(x, y, atol=1e-9) for y in uniq):
            uniq.append(x)
    return uniq


def optimum(A, b, c, l, u):
    V = vertices(A, b, l, u)
    objs = np.array([c @ v for v in V])
    best = objs.min()
    opt_vertices = [v for v, o in zip(V, objs) if o <= best + 1e-9 * (1 + abs(best))]
    return best, opt_vertices, V
