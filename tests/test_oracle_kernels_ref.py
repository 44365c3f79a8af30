"""Pins for oracle/kernels_ref.py attn_ref: against torch's SDPA (a library routine) with
a boolean mask built by an independent recursive ancestor computation + depth window,
and against the oracle model's per-beam attention over the beam's own sequence rows."""
import numpy as np
import pytest
import torch

import synth
from oracle.kernels_ref import attn_ref, build_tries


def _anc(parent, n):
    out = set()
    while n != -1:
        out.add(n)
        n = parent[n]
    return out


@pytest.mark.parametrize("Hq,Hkv,D,b,W", [(4, 4, 16, 3, 0), (8, 2, 32, 5, 0), (4, 1, 16, 4, 6),
                                          (6, 3, 8, 2, 1), (4, 2, 16, 6, 40)])
def test_attn_ref_vs_sdpa(Hq, Hkv, D, b, W):
    t = 11
    sels = [(p[None], k[None]) for p, k in synth.selections(Hq + b, 9, b, 100, 0.5)]
    T = build_tries([list(range(t))], [t], sels, b, g=2)[0]
    N = T.N
    q = synth.normal(1, 1, (b, Hq, D))
    K = synth.normal(1, 2, (Hkv, N, D))
    V = synth.normal(1, 3, (Hkv, N, D))
    o, lse = attn_ref(q, K, V, T, window=W)
    g = Hq // Hkv
    for r, leaf in enumerate(T.leaves):
        allow = _anc(T.parent, leaf)
        if W > 0:
            allow = {n for n in allow if T.depth[n] >= T.depth[leaf] - W + 1}
        mask = torch.zeros(N, dtype=torch.bool)
        mask[sorted(allow)] = True
        for h in range(Hq):
            ref = torch.nn.functional.scaled_dot_product_attention(
                torch.from_numpy(q[r, h])[None, None], torch.from_numpy(K[h // g])[None],
                torch.from_numpy(V[h // g])[None], attn_mask=mask[None, None])[0, 0].numpy()
            np.testing.assert_allclose(o[r, h], ref, atol=1e-12)
            s = K[h // g][sorted(allow)] @ q[r, h] / np.sqrt(D)
            assert abs(lse[r, h] - np.logaddexp.reduce(s)) < 1e-12
