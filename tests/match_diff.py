"""P5 match-set difference classifier -- test
infrastructure only.

The reference matches its own descriptors A_ref, B_ref; the B200 path matches
its descriptors A_gpu, B_gpu (P3 makes that match bit-equal to the reference's
matcher run on A_gpu, B_gpu).  So every pair in the symmetric difference of the
two match sets comes from the descriptor perturbation alone.  With
e_a[i] = ||A_gpu[i] - A_ref[i]|| and e_b[j] likewise, the triangle inequality
gives |D_gpu[i,j] - D_ref[i,j]| <= e_a[i] + e_b[j] for every (i, j).  A pair
(i, j) enters or leaves the mutual-nearest-neighbour set (matcher.py:74-79)
only when one of its three conditions flips:

* row i's nearest column: |D_ref[i,j] - min_{j'!=j} D_ref[i,j']| <= 2 e_a[i] + e_b[j] + max e_b
* column j's nearest row: |D_ref[i,j] - min_{i'!=i} D_ref[i',j]| <= 2 e_b[j] + e_a[i] + max e_a
* the threshold:          |D_ref[i,j] - delta_s|                  <= e_a[i] + e_b[j]

A differing pair satisfying none of them is NOT explained by a near-tie: it
is counted in ``others``, which the P5 tests require to be 0.
"""

from __future__ import annotations

import numpy as np

from oracle import lpsift_oracle as O

SLACK = 1e-12  # the float64 distance's own rounding (|D| <= 2, ~1e-15 relative)


def _second_min(D, axis):
    if D.shape[axis] < 2:
        return np.full(D.shape[1 - axis], np.inf)
    return np.partition(D, 1, axis=axis).take(1, axis=axis)


def ref_match_with_gaps(A, B, delta_s=0.35):
    """The oracle's nearest_neighbor match of (A, B) plus per-row and
    per-column (min, argmin, second-min) of the reference distance matrix, in
    one pass over O.distances (same bits as O.match)."""
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    n1, n2 = len(A), len(B)
    r_min = np.empty(n1)
    r_arg = np.empty(n1, np.int64)
    r_min2 = np.empty(n1)
    c_min = np.full(n2, np.inf)
    c_arg = np.zeros(n2, np.int64)
    c_min2 = np.full(n2, np.inf)
    for i0, D in O.distances(A, B):
        rows = np.arange(D.shape[0])
        j = np.argmin(D, axis=1)
        r_arg[i0:i0 + len(rows)] = j
        r_min[i0:i0 + len(rows)] = D[rows, j]
        r_min2[i0:i0 + len(rows)] = _second_min(D, 1)
        ci = np.argmin(D, axis=0)
        cv = D[ci, np.arange(n2)]
        cv2 = _second_min(D, 0)
        new2 = np.minimum(np.maximum(c_min, cv), np.minimum(c_min2, cv2))
        upd = cv < c_min  # strict: earlier rows win ties (first argmin)
        c_arg[upd] = ci[upd] + i0
        c_min = np.minimum(c_min, cv)
        c_min2 = new2
    rows = np.arange(n1)
    ok = (c_arg[r_arg] == rows) & (r_min < delta_s)
    r1, r2, dl = rows[ok], r_arg[ok], r_min[ok]
    order = np.lexsort((r2, r1, dl))
    stats = dict(r_min=r_min, r_arg=r_arg, r_min2=r_min2, c_min=c_min, c_arg=c_arg, c_min2=c_min2)
    return (r1[order], r2[order], dl[order]), stats


def classify(A_ref, B_ref, A_gpu, B_gpu, want, got, delta_s=0.35, stats=None):
    """Classify every pair of ``want ^ got`` (sets of (i, j)).

    Returns dict(diff, row_tie, col_tie, threshold, others, worst) where
    ``others`` lists the pairs no near-tie explains."""
    A_ref = np.asarray(A_ref, np.float64)
    B_ref = np.asarray(B_ref, np.float64)
    ea = np.linalg.norm(np.asarray(A_gpu, np.float64) - A_ref, axis=1)
    eb = np.linalg.norm(np.asarray(B_gpu, np.float64) - B_ref, axis=1)
    if stats is None:
        _, stats = ref_match_with_gaps(A_ref, B_ref, delta_s)
    ea_max = float(ea.max()) if len(ea) else 0.0
    eb_max = float(eb.max()) if len(eb) else 0.0
    out = dict(diff=0, row_tie=0, col_tie=0, threshold=0, others=[], worst=0.0)
    for (i, j) in sorted(set(want) ^ set(got)):
        out["diff"] += 1
        d = float(np.sqrt(np.sum((B_ref[j] - A_ref[i]) ** 2)))
        row_other = stats["r_min2"][i] if stats["r_arg"][i] == j else stats["r_min"][i]
        col_other = stats["c_min2"][j] if stats["c_arg"][j] == i else stats["c_min"][j]
        gaps = (
            ("row_tie", abs(d - row_other), 2 * ea[i] + eb[j] + eb_max),
            ("col_tie", abs(d - col_other), 2 * eb[j] + ea[i] + ea_max),
            ("threshold", abs(d - delta_s), ea[i] + eb[j]),
        )
        for name, gap, bound in gaps:
            if gap <= bound + SLACK:
                out[name] += 1
                out["worst"] = max(out["worst"], gap)
                break
        else:
            out["others"].append((int(i), int(j), [float(g) for _, g, _ in gaps]))
    return out
