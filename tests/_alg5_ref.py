"""Independent numpy re-derivations used to pin the oracle and to check the GPU's candidate sets.

Nothing here calls the oracle's range query, driver or bound code: the per-point region lower
bound is written out from Fig. `dist` with the AMB-7 unbounded outer regions, the
range query of Alg. 3 is a brute-force scan of the per-point predicate (AMB-12: the
result does not depend on the tree), RELAXED (Sec. 6.2.2(1)) is "every point of a leaf
whose box lower bound is <= rho" taken over an exported tree's leaves, and Alg. 5 is
re-run tree by tree (budget test after each tree, line 7; radius test after the round,
line 9).  Inputs (projections, codes, breakpoints, trees) come from whichever side is
being checked.
"""
import math

import numpy as np


def _interval(B_i, lo, hi, N_r):
    """Per-dim region interval [l, u] of symbols lo..hi (AMB-7: region 0 starts at -inf, region
    N_r - 1 ends at +inf).  B_i: [K][N_r + 1] fp64, lo/hi: [m][K] int."""
    rows = np.arange(B_i.shape[0])
    l = np.where(lo >= 1, B_i[rows, lo], -np.inf)
    u = np.where(hi <= N_r - 2, B_i[rows, np.minimum(hi + 1, N_r)], np.inf)
    return l, u


def box_lb2(B_i, lo, hi, x, N_r):
    """Squared lower bound of q' (x, [K]) to the boxes [lo, hi] ([m][K] symbols), summed over
    j in ascending order in fp64."""
    l, u = _interval(np.asarray(B_i, np.float64), np.asarray(lo, np.int64), np.asarray(hi, np.int64), N_r)
    x = np.asarray(x, np.float64)
    t = np.maximum(0.0, np.maximum(l - x, x - u))
    s = np.zeros(t.shape[0])
    for j in range(t.shape[1]):
        s += t[:, j] * t[:, j]
    return s


def cell_lb2(B_i, codes_i, x, N_r):
    """Each point's own-region lower bound (AMB-12 CELL predicate), squared."""
    return box_lb2(B_i, codes_i, codes_i, x, N_r)


class Space:
    """One side's ingredients for tree i: breakpoints B[LK][N_r+1], codes[n][LK], K, N_r."""

    def __init__(self, B, codes, K, N_r):
        self.B = np.asarray(B, np.float64)
        self.codes = np.asarray(codes)
        self.K, self.N_r = K, N_r
        self.L = self.codes.shape[1] // K

    def cell2(self, i, qp):
        sl = slice(i * self.K, (i + 1) * self.K)
        return cell_lb2(self.B[sl], self.codes[:, sl], np.asarray(qp, np.float64)[sl], self.N_r)


def radii(r_min, c, rounds):
    """r of rounds 1..rounds by repeated multiplication in double (AMB-19)."""
    out, r = [], r_min
    for _ in range(rounds):
        out.append(r)
        r = c * r
    return out


def alg5(sp: Space, eps, X, q, qp, k, c, r_min, beta, n, max_rounds=64):
    """Alg. 5, tree-granular, CELL predicate by brute-force scan.  Returns the stop (reason,
    rounds, trees_last, r_final), |S|, the final S (ascending local ids) and the top-k by
    (d^2, id) with d^2 in fp64."""
    budget = math.ceil(beta * n) + k
    cell = [sp.cell2(i, qp) for i in range(sp.L)]
    inS = np.zeros(n, bool)
    d2 = ((X.astype(np.float64) - np.asarray(q, np.float64)) ** 2).sum(1)
    r = r_min
    rounds = 0
    while True:
        rounds += 1
        stop = None
        for i in range(sp.L):
            inS |= cell[i] <= (eps * r) * (eps * r)
            if inS.sum() >= budget:
                stop = (0, i + 1)
                break
        if stop is None:
            if np.sum(d2[inS] <= (c * r) * (c * r)) >= k:
                stop = (1, sp.L)
            elif rounds == max_rounds:
                stop = (2, sp.L)
        if stop is not None:
            break
        r = c * r
    S = np.flatnonzero(inS)
    order = np.lexsort((S, d2[S]))[:k]
    return {"reason": stop[0], "rounds": rounds, "trees_last": stop[1], "r_final": r, "n_cand": len(S),
            "S": S, "ids": S[order], "d2": d2[S][order]}


def relaxed_range(tree, B_i, qp_i, rho, N_r):
    """Sec. 6.2.2(1): every point of each leaf whose (prefix) box lower bound is <= rho."""
    lb2 = box_lb2(B_i, tree["lo"], tree["hi"], qp_i, N_r)
    off = tree["leaf_off"]
    keep = np.flatnonzero(lb2 <= rho * rho)
    if len(keep) == 0:
        return np.zeros(0, np.int64)
    return np.sort(np.concatenate([tree["perm"][off[l]:off[l + 1]] for l in keep]))


def S_from_stop(sp: Space, eps, qp, r_min, c, rounds, trees_last):
    """The candidate set Alg. 5 holds when it stops in round `rounds` after tree `trees_last`:
    the union of the CELL range queries of every earlier round (radius-monotone, so the last
    full round suffices) and of the last round's first trees_last trees."""
    rs = radii(r_min, c, rounds)
    inS = np.zeros(sp.codes.shape[0], bool)
    for i in range(sp.L):
        cell = sp.cell2(i, qp)
        if i < trees_last:
            inS |= cell <= (eps * rs[-1]) ** 2
        elif rounds >= 2:
            inS |= cell <= (eps * rs[-2]) ** 2
    return inS
