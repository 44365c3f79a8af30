"""GPU vs oracle, integer path, bit-exact and teacher-forced (SURVEY §8(c) parity protocol):
trie_append (update_trie + update_mask) and trie_prune_compact (GC: mark, prune, stable
compaction, parent/leaf remap, KV row moves) against oracle.kernels_ref.build_tries on
identical selection sequences.  Compared after EVERY step: N, token, parent, depth,
beam_mask (generated nodes), leaves, and the identity of the K/V bytes in every slot."""
import numpy as np
import pytest
import torch

import synth
from oracle.kernels_ref import build_tries, soa
from tests.gpu_util import need_gpu, per_request_selections

pytestmark = pytest.mark.gpu


def _ident(depth, token, l, h, kind):
    # exact in fp32/bf16? use fp32 pools: depth*1000 + token < 2^24
    return depth * 1000.0 + token, l * 100.0 + h * 2.0 + kind


CASES = [
    # R, b, t_max, ragged, steps, rho, g
    (3, 3, 8, False, 16, 0.5, 1),
    (4, 1, 5, False, 10, 0.0, 1),
    (5, 8, 20, True, 24, 0.5, 1),
    (2, 32, 40, False, 20, 0.9, 1),
    (3, 4, 12, True, 30, 0.0, 3),
    (2, 16, 600, False, 12, 0.3, 1),   # > 512 generated+prompt rows: multi-batch scan
    (1, 32, 9, False, 40, 0.0, 1),     # 40*32 = 1280 appended nodes: multi-batch scan
    (3, 5, 7, True, 15, 1.0, 4),
]


PAGED_CASES = [CASES[0], CASES[2], CASES[4], CASES[5], CASES[7]]


def _check_pages(st, N, R, tag):
    """Paged pools (NEXT-2): request r maps exactly blocks [0, ceil(N_r / 64)); the mapped
    pages are distinct across requests; the prompt keeps its fixed pages; the device
    in-use count equals the mapped pages."""
    pt = st.page_table.cpu().numpy()
    seen = []
    for r in range(R):
        nb = (int(N[r]) + 63) // 64
        assert np.all(pt[r, :nb] >= 0) and np.all(pt[r, nb:] == -1), f"{tag} r {r}: mapped blocks"
        pp = st.prompt_pages(r)
        assert pt[r, : len(pp)].tolist() == pp, f"{tag} r {r}: prompt pages moved"
        seen += pt[r, :nb].tolist()
    assert len(seen) == len(set(seen)) and max(seen) < st.n_pages, f"{tag}: a page mapped twice"
    ps = st.page_stats()
    assert ps["in_use"] == len(seen) and ps["peak"] >= len(seen), f"{tag}: {ps} vs {len(seen)}"


@pytest.mark.parametrize("paged", [False, True], ids=["dense", "paged"])
@pytest.mark.parametrize("R,b,t_max,ragged,steps,rho,g", CASES)
def test_append_prune_bit_exact(R, b, t_max, ragged, steps, rho, g, paged):
    need_gpu()
    from paper_2502_00085_b200.trie import TrieState
    if paged and (R, b, t_max, ragged, steps, rho, g) not in PAGED_CASES:
        pytest.skip("paged pools: a subset of the cases")
    seed = R * 100 + b
    V = 1000
    lens = synth.ragged_lens(seed, R, t_max) if ragged else None
    prompts, lens = synth.prompts(seed, R, t_max, V, lens)
    sels = per_request_selections(seed, R, steps, b, V, rho)
    cap = t_max + b * steps + b
    if paged:  # NEXT-2: 64-slot pages; enough for the no-GC worst case of every request
        cap = (cap + 63) // 64 * 64
    L, Hkv, D = 2, 2, 16
    st = TrieState(R, b, t_max, cap, L, 2 * Hkv, Hkv, D, V, prompts, lens, dtype=torch.float32,
                   n_pages=R * cap // 64 if paged else 0)
    kp, vp = st.new_pools()

    def write_kv(slots_per_req):
        pt = st.page_table.cpu().numpy() if paged else None
        for r, slots in enumerate(slots_per_req):
            for n in slots:
                dep, tok = int(st.depth[r, n]), int(st.token[r, n])
                for l in range(L):
                    for h in range(Hkv):
                        for kind, pool in ((0, kp), (1, vp)):
                            a, bb = _ident(dep, tok, l, h, kind)
                            if paged:
                                pool[l, int(pt[r, n // 64]), h, n % 64, 0] = a
                                pool[l, int(pt[r, n // 64]), h, n % 64, 1] = bb
                            else:
                                pool[l, r, h, n, 0] = a
                                pool[l, r, h, n, 1] = bb

    write_kv([range(int(lens[r])) for r in range(R)])  # prompt prefill
    for k, (par, tok) in enumerate(sels, 1):
        st.append(torch.as_tensor(par, device="cuda"), torch.as_tensor(tok, device="cuda"))
        if (t_max + k) % g == 0:
            st.prune_compact(kp, vp)
        torch.cuda.synchronize()
        ref = soa(build_tries(prompts, lens, sels[:k], b, g=g, final_gc=True, t_sched=t_max), cap, b)
        N = st.n_nodes.cpu().numpy()
        assert np.array_equal(N, ref["N"]), f"step {k}: N {N} vs {ref['N']}"
        if paged:
            _check_pages(st, N, R, f"step {k}")
            kd = torch.stack([st.dense_view(kp[l]) for l in range(L)])
            vd = torch.stack([st.dense_view(vp[l]) for l in range(L)])
        else:
            kd, vd = kp, vp
        tokg, parg, depg = st.token.cpu().numpy(), st.parent.cpu().numpy(), st.depth.cpu().numpy()
        maskg = st.beam_mask.cpu().numpy().view(np.uint32)
        leafg = st.leaf.cpu().numpy()[:, :b]
        for r in range(R):
            n, t = N[r], int(lens[r])
            assert np.array_equal(tokg[r, :n], ref["token"][r, :n]), f"step {k} r {r} token"
            assert np.array_equal(parg[r, :n], ref["parent"][r, :n]), f"step {k} r {r} parent"
            assert np.array_equal(depg[r, :n], ref["depth"][r, :n]), f"step {k} r {r} depth"
            assert np.array_equal(maskg[r, t:n], ref["mask"][r, t:n]), f"step {k} r {r} mask"
            assert np.array_equal(leafg[r], ref["leaf"][r]), f"step {k} r {r} leaf"
            # leaves are the last b slots and share depth t + k - 1 (invariant 2)
            assert np.array_equal(leafg[r], np.arange(n - b, n))
            # KV identity of every slot that holds K/V (all but the pending leaves)
            kpn = kd[:, r, :, : n - b, :2].cpu().numpy()
            vpn = vd[:, r, :, : n - b, :2].cpu().numpy()
            for l in range(L):
                for h in range(Hkv):
                    exp0 = ref["depth"][r, : n - b] * 1000.0 + ref["token"][r, : n - b]
                    assert np.array_equal(kpn[l, h, :, 0], exp0), f"step {k} r {r} K rows moved wrong"
                    assert np.array_equal(vpn[l, h, :, 0], exp0)
                    assert np.all(kpn[l, h, :, 1] == l * 100.0 + h * 2.0)
                    assert np.all(vpn[l, h, :, 1] == l * 100.0 + h * 2.0 + 1)
        # forward of the new leaves: their K/V arrive now (write-before-read)
        write_kv([range(N[r] - b, N[r]) for r in range(R)])
    assert st.status() == 0


def test_capacity_overflow_latches_status():
    need_gpu()
    from paper_2502_00085_b200.trie import TrieState
    from paper_2502_00085_b200._lib import TRIE_ST_CAPACITY
    prompts, lens = synth.prompts(1, 1, 4, 50)
    st = TrieState(1, 4, 4, 12, 0, 1, 1, 16, 50, prompts, lens, dtype=torch.float32)
    par = torch.zeros(1, 4, dtype=torch.int32, device="cuda")
    tok = torch.arange(4, dtype=torch.int32, device="cuda")[None]
    st.append(par, tok)          # N = 8
    st.append(par, tok)          # N = 12 == capacity
    st.append(par, tok)          # would be 16 > 12
    assert st.status() & TRIE_ST_CAPACITY
    assert int(st.n_nodes[0]) == 12


def test_empty_prompt_rejected():
    need_gpu()
    from paper_2502_00085_b200._lib import TrieError
    from paper_2502_00085_b200.trie import TrieState
    with pytest.raises(TrieError):
        TrieState(2, 2, 4, 20, 0, 1, 1, 16, 50, np.zeros((2, 4), np.int32), [3, 0], dtype=torch.float32)


def test_paged_pool_exhaustion_latches_and_gc_returns_pages():
    """NEXT-2: with too few pages the append latches TRIE_ST_CAPACITY; with just enough,
    pruning returns pages that later appends reuse (in-use never exceeds the pool)."""
    need_gpu()
    from paper_2502_00085_b200._lib import TRIE_ST_CAPACITY
    from paper_2502_00085_b200.trie import TrieState
    prompts, lens = synth.prompts(3, 2, 60, 50)
    # 2 prompt pages + 1 free page: the second 64-slot block of both requests cannot map
    st = TrieState(2, 4, 60, 256, 0, 1, 1, 16, 50, prompts, lens, dtype=torch.float32, n_pages=3)
    par = torch.zeros(2, 4, dtype=torch.int32, device="cuda")
    tok = torch.arange(4, dtype=torch.int32, device="cuda")[None].repeat(2, 1)
    st.append(par, tok)  # N = 64: still the prompt pages
    st.append(par, tok)  # N = 68: both need a second page, one is free
    assert st.status() & TRIE_ST_CAPACITY
    # convergent chain (every new beam continues beam 0): GC keeps t + k + b - 1 rows, so
    # the pages in use stay bounded while 40 steps append 160 rows per request
    st2 = TrieState(1, 4, 60, 256, 0, 1, 1, 16, 50, prompts[:1], lens[:1], dtype=torch.float32, n_pages=3)
    for k in range(40):
        st2.append(par[:1], (tok[:1] + 4 * k) % 50)
        st2.prune_compact([], [])
    assert st2.status() == 0
    N = int(st2.n_nodes[0])
    assert N == 60 + 40 + 3
    ps = st2.page_stats()
    assert ps["in_use"] == (N + 63) // 64 and ps["peak"] <= 3
