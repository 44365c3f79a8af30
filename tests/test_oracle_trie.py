"""Pins for oracle/trie.py (Alg. 3 mask, update_trie/update_mask, §3.5 GC) and the
kernel-level packing in oracle/kernels_ref.py: SPEC worked examples, the paper's Fig. 1
counts, brute-force ancestor sets on random tries, closed-form node counts."""
import json
import os

import numpy as np
import pytest

import synth
from oracle.kernels_ref import build_tries, mask_bits, soa
from oracle.trie import (Trie, build_mask, garbage_collect, gc_mark, gc_prune_compact,
                         unique_prefix_count, update_mask, window_allow)


def _ancestors_recursive(parent, n):
    """Independent brute force: anc-or-self by recursion."""
    return {n} if parent[n] == -1 else {n} | _ancestors_recursive(parent, parent[n])


def _random_trie(seed, t, steps, b, rho):
    T = Trie(list(range(t)))
    sels = synth.selections(seed, steps, b, 50, rho)
    for par, tok in sels:
        T.update_trie([(0.0, int(tok[i]), int(par[i])) for i in range(b)])
    return T


@pytest.fixture(scope="module")
def ex(golden_dir):
    return json.load(open(os.path.join(golden_dir, "spec_worked_examples.json")))


def test_initialize_trie_examples():
    T = Trie([7, 3, 9])
    assert T.depth == [0, 1, 2] and T.leaves == [2] and T.parent == [-1, 0, 1]
    assert Trie([5]).leaves == [0]
    with pytest.raises(ValueError):
        Trie([])


def test_mask_rows_spec_example(ex):
    """t=2, leaves n2, n3 children of the last prompt node -> [T,T,T,F], [T,T,F,T]."""
    T = Trie([1, 2])
    T.update_trie([(0.0, 5, 0), (0.0, 6, 0)])
    assert build_mask(T).tolist() == ex["mask_rows"]["rows"]


def test_mask_chain_allows_everything():
    T = Trie([1, 2, 3])
    for k in range(4):
        T.update_trie([(0.0, k, 0)])
    assert build_mask(T).all()


@pytest.mark.parametrize("seed", range(1000))
def test_mask_fuzz_vs_recursive_ancestors(seed):
    """S:585 acceptance 4: 1,000 random tries (<= 64 nodes) vs the recursive oracle;
    build == update-chain; no all-false row."""
    b = 1 + seed % 5
    t = 1 + seed % 7
    steps = max(1, (64 - t) // b)
    T = Trie(list(range(t)))
    M = build_mask(T)
    sels = synth.selections(seed, steps, b, 40, rho=(seed % 10) / 10)
    for par, tok in sels:
        sel = [(0.0, int(tok[i]), int(par[i])) for i in range(b)]
        T.update_trie(sel)
        M = update_mask(M, T, sel)
        if seed % 3 == 0:
            garbage_collect(T)
            M = build_mask(T)
    Mb = build_mask(T)
    assert np.array_equal(M, Mb)
    for r, leaf in enumerate(T.leaves):
        anc = _ancestors_recursive(T.parent, leaf) | set(range(T.t))
        assert set(np.nonzero(Mb[r])[0].tolist()) == anc
    assert Mb.any(axis=1).all()


def test_swa_chain_example(ex):
    """chain of 6, window 3, leaf at position 5 -> positions {3,4,5}."""
    T = Trie(list(range(6)))
    row = window_allow(T, 5, build_mask(T)[0], 3)
    assert np.nonzero(row)[0].tolist() == ex["swa_chain"]["allowed_positions"]
    assert window_allow(T, 5, build_mask(T)[0], 1).sum() == 1        # W=1: self only
    assert window_allow(T, 5, build_mask(T)[0], 6).all()            # W >= depth+1: dense


def test_gc_mark_example(ex):
    """prompt p0,p1; n2,n3 children of p1; n4 child of n2; live leaf {n4} -> {n3}."""
    T = Trie([0, 1])
    T.update_trie([(0.0, 2, 0), (0.0, 3, 0)])   # n2, n3
    T.update_trie([(0.0, 4, 0)])                # n4 under n2 (beam 0)
    assert gc_mark(T) == {3}


def test_compact_remap_example(ex):
    """occupied {0..4}, retained [0,1,2,4] -> {0->0,1->1,2->2,4->3}."""
    T = Trie([0, 1, 2])
    T.update_trie([(0.0, 3, 0), (0.0, 4, 0)])   # slots 3, 4
    T.leaves = [4]                               # only slot 4 live
    remap = gc_prune_compact(T, gc_mark(T))
    assert {str(k): v for k, v in remap.items()} == ex["compact"]["remap"]
    assert T.parent == [-1, 0, 1, 2] and T.leaves == [3]


def test_gc_idempotent_and_conservation():
    for seed in range(50):
        T = _random_trie(seed, 5, 12, 4, 0.5)
        before = T.N
        marked = gc_mark(T)
        garbage_collect(T)
        assert T.N == before - len(marked)
        assert gc_mark(T) == set()              # S:499 mark∘prune idempotent
        # retained = U anc-or-self(leaves) ∪ prompt, exactly
        keep = set(range(T.t))
        for leaf in T.leaves:
            keep |= _ancestors_recursive(T.parent, leaf)
        assert keep == set(range(T.N))


def test_positions_match_conventional_sequence():
    """§3.4: a node's position = its index in its own beam's sequence."""
    for seed in range(20):
        T = _random_trie(seed, 4, 9, 3, 0.3)
        garbage_collect(T)
        for leaf in T.leaves:
            path = T.path(leaf)
            assert [T.depth[n] for n in path] == list(range(len(path)))


def test_unique_prefix_invariant_and_closed_forms():
    for seed in range(30):
        b, t, s = 3 + seed % 4, 6, 10
        T = Trie(list(range(t)))
        for k, (par, tok) in enumerate(synth.selections(seed, s, b, 1000, 0.5), 1):
            T.update_trie([(0.0, int(tok[i]), int(par[i])) for i in range(b)])
            assert T.N == t + b * k if k == 1 else True
        no_gc = T.N
        assert no_gc == t + b * s                  # closed form without GC
        garbage_collect(T)
        assert T.N == unique_prefix_count(T)       # BJ unique-prefix invariant
        assert t + s + b - 1 <= T.N <= t + b * s   # fully convergent lower bound


def test_fully_convergent_count():
    """Every step expands rank-0's parent only -> t + s + b - 1 nodes after GC."""
    t, s, b = 5, 7, 4
    T = Trie(list(range(t)))
    for k in range(s):
        T.update_trie([(0.0, i, 0) for i in range(b)])
        garbage_collect(T)
    assert T.N == t + s + b - 1


def test_fig1_counts(golden_dir):
    """12 trie tokens vs 21 batch tokens, under reading A17 (golden fixture)."""
    g = json.load(open(os.path.join(golden_dir, "paper_fig1_counts.json")))
    b, t = g["b"], g["t"]
    tries = build_tries([list(range(t))], [t],
                        [(np.array([p]), np.array([[10 * k + i for i in range(b)]]))
                         for k, p in enumerate(g["step_parents"])], b, g=1, final_gc=True)
    assert tries[0].N == g["trie_entries"]
    assert b * (t + g["s"]) == g["batch_entries"]
    sp = g["spec_reading"]
    for seed in range(100):  # SPEC reading: t=5, s=2 -> batch 21, trie <= 12 for any pattern
        T = build_tries([list(range(sp["t"]))], [sp["t"]],
                        [(p[None], k[None]) for p, k in synth.selections(seed, sp["s"], 3, 50, 0.5)],
                        3, g=1)[0]
        assert T.N <= sp["trie_max"]
    assert 3 * (sp["t"] + sp["s"]) == sp["batch_entries"]


def test_soa_packing_roundtrip():
    prompts_, lens = synth.prompts(3, 3, 9, 100, lens=[9, 4, 1])
    sels = [(np.stack([p] * 3), np.stack([k] * 3)) for p, k in synth.selections(3, 6, 4, 100, 0.4)]
    tries = build_tries(prompts_, lens, sels, 4, g=1)
    S = soa(tries, 64, 4)
    for r, T in enumerate(tries):
        n = T.N
        assert S["N"][r] == n
        w = S["mask"][r]
        for i, leaf in enumerate(T.leaves):
            anc = _ancestors_recursive(T.parent, leaf)
            for m in range(T.t, n):
                assert bool((w[m] >> i) & 1) == (m in anc)
        assert mask_bits(T)[: T.t].sum() == 0
