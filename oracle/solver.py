"""Oracle of the quantization-scheme solver -- plain numpy, fp64.

TEST INFRASTRUCTURE ONLY (same rule as the rest of oracle/: only tests/, smoke() and
bench.py's CPU legs may import it).  It shares no code with the library's solver
(paper_2207_04658_b200/csrc/solver.cu).

What it computes, in the paper's notation (P:n = PAPER.md line n, S:n = SPEC.md line n):
  - predict_error: Eq. 8, E[dz] = 1/12 sum_h Delta_h^2 g_h, sigma_pred =
    sqrt(E[dz]);
  - solve_error_bounded: the Lagrange solution of Eq. 9,
    Delta_h = sqrt(12 P_h (eps z)^2 / (g_h sum_h P_h)), then Algorithm 1 line 15
    (P:391): b_h = ceil(-log2(Delta_h / R_h)), clamped to [b_min, b_max]; a quantity
    with g_h = 0 does not enter the error and gets b_min;
  - solve_memory_bounded: Eq. 7, min E[dz] s.t. sum_h P_h b_h <= B.  The
    paper defers the closed form to its unavailable supplement; S:342 derives
    the stationarity solution Delta_h = c sqrt(P_h / g_h),
    log2 c = [sum_h P_h (log2 R_h - 1/2 log2(P_h / g_h)) - B] / sum_h P_h,
    then b_h = floor(-log2(Delta_h / R_h)) (floor keeps the budget hard);
  - the exhaustive integer searches the pins compare against (small H only).
B counts FRACTION bits; the stored width of a fixed field is b + 1 (sign, reading Q2),
so a budget eps_mem * M in physical bits is B = eps_mem * M - sum_h P_h.
"""
from __future__ import annotations

import itertools

import numpy as np


def predict_error(delta, g):
    """sigma_pred = sqrt(1/12 sum_h Delta_h^2 g_h) (Eq. 8)."""
    delta = np.asarray(delta, np.float64)
    g = np.asarray(g, np.float64)
    return float(np.sqrt(np.sum(delta * delta * g) / 12.0))


def error_bounded_delta(P, g, z, eps):
    """Delta_h = sqrt(12 P_h (eps z)^2 / (g_h sum P)); inf where g_h = 0."""
    P = np.asarray(P, np.float64)
    g = np.asarray(g, np.float64)
    with np.errstate(divide="ignore"):
        return np.sqrt(12.0 * P * (eps * z) ** 2 / (g * P.sum()))


def solve_error_bounded(P, g, R, z, eps, b_min=0, b_max=31):
    """Algorithm 1 lines 13-15.  Returns (Delta_h, b_h)."""
    R = np.asarray(R, np.float64)
    g = np.asarray(g, np.float64)
    delta = error_bounded_delta(P, g, z, eps)
    bits = np.empty(len(R), np.int64)
    for h in range(len(R)):
        if g[h] == 0.0:
            bits[h] = b_min
        else:
            bits[h] = min(max(int(np.ceil(-np.log2(delta[h] / R[h]))), b_min), b_max)
    return delta, bits


def solve_memory_bounded(P, g, R, budget_bits, b_min=0, b_max=31):
    """Eq. 7 with the stationarity solution of S:342 over the box [b_min, b_max]:
    quantities with g_h = 0 take b_min; the closed form is solved over the free
    quantities with the budget the fixed ones leave, and a free quantity whose floored
    width leaves the box is fixed at the bound and the rest re-solved (active set).
    Returns (Delta_h, b_h); raises ValueError when no scheme in the box fits."""
    P = np.asarray(P, np.float64)
    g = np.asarray(g, np.float64)
    R = np.asarray(R, np.float64)
    H = len(P)
    if np.sum(P * b_min) > budget_bits:
        raise ValueError("budget below b_min everywhere")
    delta = np.full(H, np.inf)
    bits = np.full(H, b_min, np.int64)
    fixed = ~(g > 0.0)
    for _ in range(H + 1):
        free = ~fixed
        if not free.any():
            break
        B = budget_bits - np.sum(P[fixed] * bits[fixed])
        Pa, ga, Ra = P[free], g[free], R[free]
        log2c = (np.sum(Pa * (np.log2(Ra) - 0.5 * np.log2(Pa / ga))) - B) / np.sum(Pa)
        changed = False
        for h in np.nonzero(free)[0]:
            d = 2.0 ** log2c * np.sqrt(P[h] / g[h])
            b = np.floor(-np.log2(d / R[h]))
            delta[h] = d
            bits[h] = min(max(int(b), b_min), b_max)
            if b < b_min or b > b_max:
                fixed[h] = True
                changed = True
        if not changed:
            break
    if np.sum(P * bits) > budget_bits * (1.0 + 1e-12):
        raise ValueError("no scheme within [b_min, b_max] fits the budget")
    return delta, bits


def bits_to_delta(bits, R):
    """Delta = R 2^-b."""
    return np.asarray(R, np.float64) * 2.0 ** (-np.asarray(bits, np.float64))


def brute_force_error_bounded(P, g, R, z, eps, b_max=20):
    """Exhaustive: the integer bit vector minimising sum P_h b_h subject to
    sigma_pred <= eps |z| (small H only)."""
    best = None
    for b in itertools.product(range(b_max + 1), repeat=len(P)):
        if predict_error(bits_to_delta(b, R), g) <= eps * abs(z):
            cost = float(np.dot(P, b))
            if best is None or cost < best[0]:
                best = (cost, np.array(b))
    return best


def brute_force_memory_bounded(P, g, R, budget_bits, b_max=20):
    """Exhaustive: the integer bit vector minimising sigma_pred subject to
    sum P_h b_h <= B (small H only)."""
    best = None
    for b in itertools.product(range(b_max + 1), repeat=len(P)):
        if float(np.dot(P, b)) <= budget_bits:
            err = predict_error(bits_to_delta(b, R), g)
            if best is None or err < best[0]:
                best = (err, np.array(b))
    return best
