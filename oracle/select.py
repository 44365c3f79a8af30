"""Global top-b beam selection (Alg. 1 l.6 "top-b" P:116; Alg. 2 l.9 "argsort_b" P:146).

Reading R1: argsort_b is the GLOBAL top-b over all (live beam j, token v)
candidates by cumulative log-probability score_j + lp_j[v].  Reading R3: the
order is total -- score descending, then token v ascending, then beam j ascending
(S:306); the new beams are returned in that rank order.  Reading R2: b' = min(b, #cand).
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np


def select_topb(scores, lp_rows, b: int):
    """scores[j] (cumulative), lp_rows[j][v] (log-probs) for the live beams j.

    Returns a list of (new_score, v, j) in rank order, length min(b, J*V).
    Plain Python sort over every candidate (obviously correct, slow).
    """
    cands = []
    for j, (s, lp) in enumerate(zip(scores, lp_rows)):
        for v in range(len(lp)):
            cands.append((s + lp[v], v, j))
    cands.sort(key=lambda c: (-c[0], c[1], c[2]))
    return cands[: min(b, len(cands))]


def select_topb_np(scores, lp_rows, b: int):
    """Same selection with a library sort (np.lexsort) for large b*V (kernel-level use).

    lexsort's primary key is the LAST key: (-score) then v then j, exactly the order of
    select_topb.  Returns (new_score[b'], v[b'], j[b']).
    """
    lp_rows = np.asarray(lp_rows)
    J, V = lp_rows.shape
    cs = (np.asarray(scores, dtype=lp_rows.dtype)[:, None] + lp_rows).reshape(-1)
    jj = np.repeat(np.arange(J), V)
    vv = np.tile(np.arange(V), J)
    order = np.lexsort((jj, vv, -cs))[: min(b, J * V)]
    return cs[order], vv[order], jj[order]
