"""End to end on the GPU, BASELINE.json configs[0]: tiny random-init 2-layer decoder
(d=64, 4 heads, V=256), prompt 8, b=3, 16 decode steps, fp32 mode (TF32 off).  The GPU
decode (model context in torch + every trie step in libtriedecode) must reproduce the
oracle's Alg. 2 trie beam search (itself pinned == Alg. 1 batch beam search): identical
tokens, parents and final hypotheses, scores within 1e-4 relative; near-ties switch to
lockstep."""
import numpy as np
import pytest
import torch

import synth
from oracle.decode import trie_beam_search
from oracle.model import Model, ModelConfig
from tests.gpu_util import need_gpu

pytestmark = pytest.mark.gpu

CASES = [
    # seed, Hkv, b, window, R, g
    (0, 4, 3, 0, 4, 1),
    (1, 2, 3, 0, 3, 1),
    (2, 4, 5, 0, 2, 1),
    (3, 4, 1, 0, 3, 1),
    (4, 4, 3, 5, 3, 1),
    (5, 2, 4, 3, 2, 1),
    (6, 4, 3, 0, 2, 4),
    (7, 1, 8, 0, 2, 1),
]


@pytest.mark.parametrize("seed,Hkv,b,W,R,g", CASES)
def test_tiny_decode_matches_oracle(seed, Hkv, b, W, R, g):
    need_gpu()
    from paper_2502_00085_b200.decode import trie_beam_decode
    from paper_2502_00085_b200.model import TinyModel
    from paper_2502_00085_b200.trie import TrieState
    t, s, V = 8, 16, 256
    prompts, lens = synth.prompts(seed, R, t, V)
    gm = TinyModel(seed, Hkv=Hkv)
    st = TrieState(R, b, t, t + b * s + b, 2, 4, Hkv, 16, V, prompts, lens, window=W,
                   gc_interval=g, dtype=torch.float32)
    kp, vp = st.new_pools()
    toks, lens_out, scores, trace = trie_beam_decode(gm, st, kp, vp, prompts, lens, s, g=g,
                                                     record=True)
    assert st.status() == 0
    om = Model(synth.tiny_weights(seed, 2, 64, 4, Hkv, 16, 256, V), ModelConfig(Hkv=Hkv))
    for r in range(R):
        ref = trie_beam_search(om, [int(x) for x in prompts[r]], b, s, g=g, window=W)
        for k, step in enumerate(ref.steps):
            sel = step["sel"]
            gp, gt = trace[k]["par"][r], trace[k]["tok"][r]
            assert [j for _, _, j in sel] == gp.tolist() and [v for _, v, _ in sel] == gt.tolist(), \
                f"r={r} step {k + 1}: GPU {list(zip(gp, gt))} vs oracle {[(j, v) for _, v, j in sel]}"
            np.testing.assert_allclose(trace[k]["score"][r], [sc for sc, _, _ in sel], rtol=1e-4, atol=1e-4)
            np.testing.assert_allclose(trace[k]["logits"][r][: len(step["lp_rows"])] -
                                       trace[k]["logits"][r][: len(step["lp_rows"])].max(-1, keepdims=True),
                                       np.stack(step["lp_rows"]) - np.stack(step["lp_rows"]).max(-1, keepdims=True),
                                       atol=2e-4)
        for j, (htoks, hsc) in enumerate(ref.hyps):
            assert lens_out[r, j] == len(htoks)
            assert toks[r, j, : len(htoks)].tolist() == htoks
            assert abs(scores[r, j] - hsc) <= 1e-4 * max(1.0, abs(hsc))



@pytest.mark.parametrize("seed,Hkv,b,R", [(0, 4, 3, 3), (7, 1, 8, 2), (2, 4, 5, 2)])
def test_tiny_decode_with_eos_matches_oracle(seed, Hkv, b, R):
    """NEXT-3 (reading R5b): EOS as an absorbing token, end to end vs the oracle.  The EOS
    id is a token the oracle selects at step 3 for request 0, so finished beams occur."""
    need_gpu()
    from paper_2502_00085_b200.decode import trie_beam_decode
    from paper_2502_00085_b200.model import TinyModel
    from paper_2502_00085_b200.trie import TrieState
    t, s, V = 8, 16, 256
    prompts, lens = synth.prompts(seed, R, t, V)
    om = Model(synth.tiny_weights(seed, 2, 64, 4, Hkv, 16, 256, V), ModelConfig(Hkv=Hkv))
    eos = trie_beam_search(om, [int(x) for x in prompts[0]], b, 4, g=1).steps[2]["sel"][0][1]
    gm = TinyModel(seed, Hkv=Hkv)
    st = TrieState(R, b, t, t + b * s + b, 2, 4, Hkv, 16, V, prompts, lens, dtype=torch.float32)
    kp, vp = st.new_pools()
    toks, lens_out, scores, trace = trie_beam_decode(gm, st, kp, vp, prompts, lens, s, g=1,
                                                     record=True, eos=eos)
    assert st.status() == 0
    fin_seen = 0
    for r in range(R):
        ref = trie_beam_search(om, [int(x) for x in prompts[r]], b, s, g=1, eos=eos)
        for k, step in enumerate(ref.steps):
            sel = step["sel"]
            gp, gt = trace[k]["par"][r], trace[k]["tok"][r]
            assert [j for _, _, j in sel] == gp.tolist() and [v for _, v, _ in sel] == gt.tolist(), \
                f"r={r} step {k + 1}: GPU {list(zip(gp, gt))} vs oracle {[(j, v) for _, v, j in sel]}"
            np.testing.assert_allclose(trace[k]["score"][r], [sc for sc, _, _ in sel], rtol=1e-4, atol=1e-4)
            fin_seen += sum(v == eos for _, v, _ in sel)
        for j, (htoks, hsc) in enumerate(ref.hyps):
            assert toks[r, j, : len(htoks)].tolist() == htoks
            assert abs(scores[r, j] - hsc) <= 1e-4 * max(1.0, abs(hsc))
        fin = st.finished.cpu().numpy()[r, :b] != 0
        assert fin.tolist() == [h[0][-1] == eos for h in ref.hyps]
    assert fin_seen > 0
