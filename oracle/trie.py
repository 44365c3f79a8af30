"""The trie T of Alg. 2, its attention mask (Alg. 3) and garbage collection (§3.5).

Slot convention (reading R10/R21): the prompt occupies slots 0..t-1 as a chain
(parent[i] = i-1, depth[i] = i); generated nodes are appended at the end, so
parent[n] < n.  Mask columns are slots 0..N-1 (the paper's t + |T| columns).

TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np


class Trie:
    """Alg. 2 l.1 initialize_trie(prompt)."""

    def __init__(self, prompt, n_layers: int = 0):
        prompt = [int(x) for x in prompt]
        if not prompt:
            raise ValueError("empty prompt (S:260)")
        self.t = len(prompt)
        self.token = list(prompt)
        self.parent = [-1] + list(range(self.t - 1))
        self.depth = list(range(self.t))  # §3.4: positions of the conventional sequence
        self.kv = [[None] * self.t for _ in range(n_layers)]  # per layer: slot -> (k, v)
        self.leaves = [self.t - 1]
        self.scores = [0.0]

    @property
    def N(self) -> int:
        return len(self.token)

    def has_kv(self, n: int) -> bool:
        return bool(self.kv) and self.kv[0][n] is not None

    # ---- Alg. 2 l.10 update_trie (§3.4) -----------------------
    def update_trie(self, sel):
        """sel = [(new_score, token v, parent beam j)] in rank order.  New node for rank r
        at slot N + r with parent = leaves[j] and depth = depth[parent] + 1 (§3.4: the
        position it has in conventional beam search).  Leaves become the new nodes."""
        new_leaves = []
        for (sc, v, j) in sel:
            p = self.leaves[j]
            self.token.append(int(v))
            self.parent.append(p)
            self.depth.append(self.depth[p] + 1)
            for lay in self.kv:
                lay.append(None)  # pending: KV computed at the next forward
            new_leaves.append(self.N - 1)
        self.leaves = new_leaves
        self.scores = [sc for (sc, _, _) in sel]

    def path(self, n: int):
        """Root-to-node slots (ancestors-or-self, ascending)."""
        out = []
        while n != -1:
            out.append(n)
            n = self.parent[n]
        return out[::-1]

    def path_tokens(self, n: int):
        return [self.token[m] for m in self.path(n)]


# ---- Alg. 3 Causal Mask Construction ----------------------------------------
def build_mask(T: Trie) -> np.ndarray:
    """Literal Alg. 3: M <- -inf (False); M[:, :t] <- 0 (True); walkers start at the
    leaves; each round every walker allows its current node and moves to its parent;
    stop when no walker moved (`reached_root`).  Returns bool [b][N]."""
    b = len(T.leaves)
    M = np.zeros((b, T.N), dtype=bool)          # l.1
    M[:, : T.t] = True                           # l.2
    V = list(T.leaves)                           # l.3
    while True:                                  # l.4
        reached_root = True                      # l.5
        for i in range(b):                       # l.6
            M[i, V[i]] = True                    # l.7  allow attention to current node
            if T.parent[V[i]] != -1:             # l.8
                V[i] = T.parent[V[i]]            # l.9  move up the tree
                reached_root = False             # l.10
        if reached_root:                         # l.13
            return M                             # l.14


def update_mask(M: np.ndarray, T: Trie, sel) -> np.ndarray:
    """Alg. 2 l.11 update_mask (§3.3): row r of the new mask is
    the row of its parent beam j_r extended by the new columns, with its own column set."""
    b_new = len(sel)
    N_old = M.shape[1]
    M2 = np.zeros((b_new, T.N), dtype=bool)
    for r, (_, _, j) in enumerate(sel):
        M2[r, :N_old] = M[j]
        M2[r, T.leaves[r]] = True
    return M2


def window_allow(T: Trie, leaf: int, row: np.ndarray, window: int) -> np.ndarray:
    """Reading R14 (SWA along the branch): additionally require
    depth[n] >= depth[leaf] - W + 1 (W keys including self); W <= 0 means dense."""
    if window <= 0:
        return row
    lo = T.depth[leaf] - window + 1
    return row & (np.asarray(T.depth) >= lo)


# ---- §3.5 Garbage collection -------------------------------------
def gc_mark(T: Trie) -> set:
    """Marking: traverse bottom-up from the leaves to the root; every node never visited
    is marked for removal.  Prompt nodes lie on every path (never marked)."""
    visited = [False] * T.N
    for leaf in T.leaves:
        n = leaf
        while n != -1 and not visited[n]:
            visited[n] = True
            n = T.parent[n]
    return {n for n in range(T.N) if not visited[n]}


def gc_prune_compact(T: Trie, marked: set) -> dict:
    """Pruning + Compaction: keep unmarked slots in ascending order (the
    index_select of the paper), move each kept row n to new[n] = #{kept m < n}, remap
    parent and leaves.  Returns the old->new remapping of kept slots."""
    retained = [n for n in range(T.N) if n not in marked]
    new = {old: i for i, old in enumerate(retained)}
    T.token = [T.token[n] for n in retained]
    T.parent = [(-1 if T.parent[n] == -1 else new[T.parent[n]]) for n in retained]
    T.depth = [T.depth[n] for n in retained]
    T.kv = [[lay[n] for n in retained] for lay in T.kv]
    T.leaves = [new[n] for n in T.leaves]
    return new


def garbage_collect(T: Trie) -> dict:
    """Alg. 2 l.6 garbage_collect(): mark -> prune -> compact."""
    return gc_prune_compact(T, gc_mark(T))


def unique_prefix_count(T: Trie) -> int:
    """Number of distinct prefixes (root-to-node token paths) of the live hypotheses,
    prompt prefixes included: |U_r anc-or-self(leaf_r)| -- the BJ unique-prefix invariant."""
    seqs = set()
    for leaf in T.leaves:
        toks = T.path_tokens(leaf)
        for k in range(1, len(toks) + 1):
            seqs.add(tuple(toks[:k]))
    return len(seqs)
