"""Kernel-level reference functions: the pure functions each GPU entry point is compared
against, expressed with the oracle's own trie operations (oracle/trie.py) and plain
numpy float64.  Outputs are packed into the structure-of-arrays layout the C ABI uses
 only at the very end, so the packing is representation, not
arithmetic.  TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np

from .numerics import log_softmax
from .select import select_topb_np
from .trie import Trie, build_mask, garbage_collect, window_allow


# ---- integer path ----------------------------------------------------------------------
def build_tries(prompts, prompt_lens, sel_seq, b: int, g=1, final_gc=True, t_sched=None):
    """Teacher-forced trie evolution for R requests: for each step k apply the given
    (parent_beam, token) selection with update_trie (Alg. 2 l.10), then GC iff
    (t + k) mod g == 0 (reading R7/R8: Alg. 2's top-of-iteration check, placed after the
    append of step k; `final_gc` also applies it after the last step).
    sel_seq[k] = (parent[R][b_k], token[R][b_k]).  t_sched (default: each request's own t)
    replaces t in the schedule test, for batched drivers that share one schedule across
    ragged prompts (GC timing never changes outputs, only when memory is reclaimed).
    Returns a list of Trie."""
    tries = []
    for r in range(len(prompt_lens)):
        T = Trie(prompts[r][: prompt_lens[r]])
        steps = len(sel_seq)
        for k, (par, tok) in enumerate(sel_seq, start=1):
            sel = [(0.0, int(tok[r][i]), int(par[r][i])) for i in range(len(par[r]))]
            T.update_trie(sel)
            last = k == steps
            tt = T.t if t_sched is None else t_sched
            if g is not None and (tt + k) % g == 0 and (final_gc or not last):
                garbage_collect(T)
        tries.append(T)
    return tries


def mask_bits(T: Trie) -> np.ndarray:
    """Alg. 3 mask of T packed per node: bit r of word n <=> M[r][n] (generated nodes
    only; words of prompt nodes are reported as 0 -- prompt columns are implicitly
    allowed for every beam)."""
    M = build_mask(T)
    words = np.zeros(T.N, dtype=np.uint32)
    for r in range(M.shape[0]):
        words |= (M[r].astype(np.uint32) << np.uint32(r))
    words[: T.t] = 0
    return words


def soa(tries, cap: int, b: int):
    """Pack tries into [R][cap] token/parent/depth/mask, [R][b] leaf, [R] N."""
    R = len(tries)
    out = dict(token=np.zeros((R, cap), np.int32), parent=np.full((R, cap), -1, np.int32),
               depth=np.zeros((R, cap), np.int32), mask=np.zeros((R, cap), np.uint32),
               leaf=np.zeros((R, b), np.int32), N=np.zeros(R, np.int32))
    for r, T in enumerate(tries):
        n = T.N
        out["token"][r, :n] = T.token
        out["parent"][r, :n] = T.parent
        out["depth"][r, :n] = T.depth
        out["mask"][r, :n] = mask_bits(T)
        out["leaf"][r, : len(T.leaves)] = T.leaves
        out["N"][r] = n
    return out


# ---- a-3 trie attention ------------------------------------------------------------------
def attn_ref(q, K, V, T: Trie, window: int = 0):
    """§3.3: o[r,h] = sum_{n in A_r} softmax_n(q[r,h].k_n / sqrt(D)) v_n with
    A_r = Alg. 3 mask row of leaf r, windowed by depth (reading R14).
    q [b][Hq][D]; K, V [Hkv][N][D] (this request, this layer).  float64.
    Returns o [b][Hq][D] and lse [b][Hq] (natural log of sum exp(scaled scores))."""
    q = np.asarray(q, np.float64)
    K = np.asarray(K, np.float64)
    V = np.asarray(V, np.float64)
    b, Hq, D = q.shape
    Hkv = K.shape[0]
    g = Hq // Hkv
    M = build_mask(T)
    o = np.zeros((b, Hq, D))
    lse = np.zeros((b, Hq))
    for r in range(b):
        leaf = T.leaves[r]
        rows = np.nonzero(window_allow(T, leaf, M[r], window))[0]
        for h in range(Hq):
            Kh = K[h // g][rows]
            s = (Kh @ q[r, h]) / np.sqrt(D)
            m = s.max()
            e = np.exp(s - m)
            l = e.sum()
            o[r, h] = (e @ V[h // g][rows]) / l
            lse[r, h] = m + np.log(l)
    return o, lse


# ---- a-4 log-softmax + global top-b ------------------------------------------------------
def beam_step_ref(logits, scores, b: int):
    """Alg. 2 l.9 argsort_b over cumulative log-probs (reading R1, R3).  logits
    [b_live][V] (any float dtype, evaluated in float64), scores [b_live].
    Returns (parent_beam, token, new_score, gap) where gap = score(rank b-1) -
    score(rank b) (inf if there is no rank b), used by the near-tie protocol."""
    lp = np.stack([log_softmax(np.asarray(x, np.float64)) for x in logits])
    J, Vv = lp.shape
    cs, vv, jj = select_topb_np(np.asarray(scores, np.float64), lp, min(b + 1, J * Vv))
    k = min(b, J * Vv)
    gap = (cs[k - 1] - cs[k]) if len(cs) > k else np.inf
    return jj[:k].astype(np.int32), vv[:k].astype(np.int32), cs[:k], gap, lp
