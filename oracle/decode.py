"""Oracle decoders: Alg. 1 batch beam search, Alg. 2 trie beam search, greedy.

Both beam decoders call the same one-token `model.forward(token, pos, ctx)` and the same
`select_topb`; they differ only in where K/V live and which rows a query reads:
  * batch (Alg. 1): every beam owns a full copy of its cache and
    reads rows 0..pos of its own sequence;
  * trie (Alg. 2): one shared slot pool; leaf r reads the slots its mask row
    allows (Alg. 3 / update_mask), in ascending slot order = ascending depth = the
    beam's sequence order, optionally windowed by depth (reading R14).
With identical per-query row lists the two are bitwise equal in float64 -- the paper's
"theoretically equivalent" claim made checkable.

Fixed new-token count s (reading R5: no EOS on the hot path), L = t + s (reading R20);
optionally EOS as an absorbing token (`eos`, reading R5b, select.absorb_eos).
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .select import absorb_eos, select_topb
from .trie import Trie, build_mask, garbage_collect, update_mask, window_allow


@dataclass
class DecodeResult:
    hyps: list                      # [(tokens incl. prompt, score)] in rank order
    best: tuple                     # rank 0 = highest cumulative log-prob
    steps: list = field(default_factory=list)  # per step: dict(sel, lp_rows, entries, ...)


# ---------------------------------------------------------------------------------------
# Alg. 1 -- batch-based beam search
# ---------------------------------------------------------------------------------------
class _Beam:
    def __init__(self, tokens, cache, score):
        self.tokens = list(tokens)
        self.cache = cache            # per layer: list of (k, v) rows in sequence order
        self.score = score


def _forward_beam(model, beam: _Beam, window: int):
    """Feed every token of `beam` that has no KV yet (the prompt at the first iteration,
    then the newest token); returns lp of the last one (Alg. 1 l.5)."""
    lp = None
    for p in range(len(beam.cache[0]), len(beam.tokens)):
        def ctx(l, k, v, p=p):
            beam.cache[l].append((k, v))
            lo = 0 if window <= 0 else max(0, p - window + 1)
            rows = beam.cache[l][lo: p + 1]
            return np.stack([r[0] for r in rows]), np.stack([r[1] for r in rows])
        lp = model.forward(beam.tokens[p], p, ctx)
    return lp


def batch_beam_search(model, prompt, b: int, s: int, window: int = 0, eos=None) -> DecodeResult:
    L_layers = model.cfg.L
    beams = [_Beam(prompt, [[] for _ in range(L_layers)], 0.0)]      # l.1-2
    res = DecodeResult(hyps=[], best=None)
    t = len(prompt)
    for i in range(t, t + s):                                          # l.3
        if eos is not None and len(beams) == b and all(
                len(bm.tokens) > t and bm.tokens[-1] == eos for bm in beams):
            break  # reading R5b: every beam finished -> decoding stops
        lp_rows = [_forward_beam(model, bm, window) for bm in beams]   # l.4-5
        fin = [len(bm.tokens) > t and bm.tokens[-1] == eos for bm in beams]
        lp_rows = absorb_eos(lp_rows, fin, eos)                        # reading R5b
        sel = select_topb([bm.score for bm in beams], lp_rows, b)      # l.6
        beams = [_Beam(beams[j].tokens + [v],
                       [list(lay) for lay in beams[j].cache],          # per-beam copy
                       sc) for (sc, v, j) in sel]
        res.steps.append(dict(sel=sel, lp_rows=lp_rows,
                              entries=sum(len(bm.tokens) for bm in beams)))
    res.hyps = [(bm.tokens, bm.score) for bm in beams]
    res.best = res.hyps[0]                                             # l.8
    return res


# ---------------------------------------------------------------------------------------
# Alg. 2 -- trie-based beam search
# ---------------------------------------------------------------------------------------
def _forward_trie(model, T: Trie, M: np.ndarray, window: int):
    """Alg. 2 l.9 model call P(x | input, M).  Serialized input = nodes without KV
    (reading R21: incremental serialization): the prompt chain at the first iteration,
    then the b leaves.  Each query writes its K/V into its own slot first."""
    pending = [n for n in range(T.N) if not T.has_kv(n)]
    lp_by_node = {}
    for n in pending:
        if n in T.leaves:
            row = M[T.leaves.index(n)]
        else:  # prompt prefill: the ancestors-or-self of n (Alg. 3 walk from n)
            row = np.zeros(T.N, dtype=bool)
            row[T.path(n)] = True
        row = window_allow(T, n, row, window)
        allowed = [m for m in range(T.N) if row[m]]          # ascending slot order

        def ctx(l, k, v, n=n, allowed=allowed):
            T.kv[l][n] = (k, v)                              # write before read
            return (np.stack([T.kv[l][m][0] for m in allowed]),
                    np.stack([T.kv[l][m][1] for m in allowed]))
        lp_by_node[n] = model.forward(T.token[n], T.depth[n], ctx)   # position = depth
    return [lp_by_node[leaf] for leaf in T.leaves]


def trie_beam_search(model, prompt, b: int, s: int, g=1, window: int = 0,
                     final_gc: bool = False, eos=None) -> DecodeResult:
    """Alg. 2.  g = GC interval (None = never, reading R7: GC at the top of
    iteration i iff i mod g == 0).  final_gc additionally collects after the last
    append (used only for counting unique prefixes of the final hypotheses)."""
    T = Trie(prompt, n_layers=model.cfg.L)                   # l.1
    M = build_mask(T)                                        # l.2
    t = T.t                                                  # l.3 serialize -> |input| = t
    res = DecodeResult(hyps=[], best=None)
    for i in range(t, t + s):                                # l.4
        if eos is not None and len(T.leaves) == b and all(
                T.depth[leaf] >= t and T.token[leaf] == eos for leaf in T.leaves):
            break  # reading R5b: every beam finished -> decoding stops
        gc_ran = False
        if g is not None and i % g == 0:                     # l.5
            garbage_collect(T)                               # l.6
            M = build_mask(T)                                # l.7
            gc_ran = True
        lp_rows = _forward_trie(model, T, M, window)         # l.9 P(x | input, M)
        fin = [T.depth[leaf] >= t and T.token[leaf] == eos for leaf in T.leaves]
        lp_rows = absorb_eos(lp_rows, fin, eos)              # reading R5b
        sel = select_topb(T.scores, lp_rows, b)              # l.9 argsort_b
        T.update_trie(sel)                                   # l.10
        M = update_mask(M, T, sel)                           # l.11
        res.steps.append(dict(sel=sel, lp_rows=lp_rows, entries=T.N, gc=gc_ran))
    if final_gc and g is not None and (t + s) % g == 0:
        garbage_collect(T)
    res.hyps = [(T.path_tokens(leaf), sc) for leaf, sc in zip(T.leaves, T.scores)]
    res.best = res.hyps[0]                                   # l.14
    res.trie = T
    return res


def greedy_decode(model, prompt, s: int) -> list:
    """Argmax per step, lowest token id on ties (P:19 greedy; Table 1 b=1 rows)."""
    bm = _Beam(prompt, [[] for _ in range(model.cfg.L)], 0.0)
    for _ in range(s):
        lp = _forward_beam(model, bm, 0)
        v = int(np.argmax(lp))        # first maximal index = lowest token id
        bm.tokens.append(v)
        bm.score += lp[v]
    return bm.tokens, bm.score
