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


def absorb_eos(lp_rows, finished, eos):
    """NEXT-3, reading R5b (the paper is silent on EOS; SPEC's retire rule binds
    only its CPU program): EOS is an ABSORBING token.  A beam whose last generated token is
    `eos` (finished[j]) has the one-hot next-token distribution at eos (log-prob 0 there,
    -inf elsewhere), so it stays a candidate with its score unchanged and keeps competing
    for the b beams.  Returns the rows to select over (the others unchanged)."""
    if eos is None:
        return lp_rows
    out = []
    for lp, fin in zip(lp_rows, finished):
        if fin:
            row = np.full(len(lp), -np.inf)
            row[eos] = 0.0
            out.append(row)
        else:
            out.append(lp)
    return out
