"""Beam-decode driver on one GPU (Alg. 2), all trie work in libtriedecode.

Per step k = 1..s:  [forward of the b_live leaves: model context + trie_rope_kv_append +
trie_attn_decode]  ->  trie_beam_step (argsort_b + update_trie + update_mask)  ->
trie_prune_compact iff (t_max + k) % g == 0  (Alg. 2 l.5: GC at the top of iteration
i = t + k, reading R7/R8; skipped after the last step unless final_gc).
"""
from __future__ import annotations

import torch


def gc_due(t: int, k: int, s: int, g, final_gc: bool) -> bool:
    if g is None or g <= 0:
        return False
    if k == s and not final_gc:
        return False
    return (t + k) % g == 0


@torch.no_grad()
def trie_beam_decode(model, st, k_pools, v_pools, prompts, lens, s, g=1, final_gc=False,
                     record=False, eos=None):
    """Returns (hyps tokens [R][b][max_len], lens [R][b], scores [R][b], trace).
    eos: token id of an absorbing end-of-sequence (trie_set_eos, NEXT-3), None = off."""
    st.set_eos(-1 if eos is None else int(eos))
    logits = model.prefill(prompts, lens, k_pools, v_pools, window=st.window)
    trace = []
    R, b = st.R, st.b
    for k in range(1, s + 1):
        sp = torch.empty(R, b, dtype=torch.int32, device=st.device)
        tk = torch.empty_like(sp)
        sc = torch.empty(R, b, dtype=torch.float32, device=st.device)
        st.beam_step(logits, sp, tk, sc)
        if gc_due(st.t_max, k, s, g, final_gc):
            st.prune_compact(k_pools, v_pools)
        if record:
            trace.append(dict(par=sp.cpu().numpy(), tok=tk.cpu().numpy(), score=sc.cpu().numpy(),
                              N=st.n_nodes.cpu().numpy().copy(), logits=logits.cpu().numpy()))
        if k < s:
            logits = model.step(st, k_pools, v_pools)
    toks, lens_out, scores = st.read_hyps(st.t_max + s)
    return toks, lens_out, scores, trace
