"""Random-init model CONTEXT around the hot path (north_star: "model GEMMs ... are context,
not product").  cuBLAS GEMMs / norms / MLP through torch; the per-step attention path
(RoPE at trie depth + KV append, trie attention) and the beam step run in libtriedecode.

The prompt prefill (a plain causal forward over the t prompt tokens) is also
context: it writes the prompt's K/V into slots 0..t-1 of the pools and returns the
logits of the last prompt token.
"""
from __future__ import annotations

import math

import numpy as np
import torch

import synth


def rms_norm(x, g, eps):
    return x * g * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps)


def rope_torch(x, pos, base):
    """Rotate-half RoPE for the prefill context (angles in fp64, reading R16)."""
    D = x.shape[-1]
    h = D // 2
    i = torch.arange(h, dtype=torch.float64, device=x.device)
    ang = pos.to(torch.float64)[:, None] * (base ** (-2.0 * i / D))[None, :]
    c = torch.cos(ang).to(torch.float32)[:, None, :]
    s = torch.sin(ang).to(torch.float32)[:, None, :]
    xf = x.float()
    x1, x2 = xf[..., :h], xf[..., h:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1).to(x.dtype)


class TinyModel:
    """The toy decoder of BASELINE.json configs[0] (L=2, d=64, 4 heads, V=256), fp32,
    TF32 disabled, weights from synth.tiny_weights (the same numbers the oracle uses)."""

    def __init__(self, seed, L=2, d=64, Hq=4, Hkv=4, D=16, ffn=256, V=256, rope_base=10000.0,
                 eps=1e-5, kappa=4.0, device="cuda", dtype=torch.float32):
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False
        w = synth.tiny_weights(seed, L, d, Hq, Hkv, D, ffn, V)
        T = lambda a: torch.as_tensor(np.asarray(a), dtype=dtype, device=device)
        self.emb, self.lm, self.gf = T(w["emb"]), T(w["lm"]), T(w["gf"])
        self.layers = [{k: T(v) for k, v in lw.items()} for lw in w["layers"]]
        self.L, self.d, self.Hq, self.Hkv, self.D, self.V = L, d, Hq, Hkv, D, V
        self.base, self.eps, self.kappa = rope_base, eps, kappa
        self.dtype = dtype

    def _mlp(self, x, lw):
        h2 = rms_norm(x, lw["g2"], self.eps)
        return x + (torch.nn.functional.silu(h2 @ lw["wg"]) * (h2 @ lw["wu"])) @ lw["wd"]

    def _logits(self, x):
        return (self.kappa * (rms_norm(x, self.gf, self.eps) @ self.lm)).float()

    @torch.no_grad()
    def prefill(self, prompts, lens, k_pools, v_pools, window=0):
        """Causal forward of each prompt; writes K/V rows 0..t-1; returns [R][1][V]."""
        R = len(lens)
        out = torch.empty(R, 1, self.V, dtype=torch.float32, device=self.emb.device)
        g = self.Hq // self.Hkv
        for r in range(R):
            t = int(lens[r])
            toks = torch.as_tensor(np.asarray(prompts[r][:t]), dtype=torch.long, device=self.emb.device)
            pos = torch.arange(t, device=self.emb.device)
            x = self.emb[toks]
            for l, lw in enumerate(self.layers):
                h = rms_norm(x, lw["g1"], self.eps)
                q = rope_torch((h @ lw["wq"]).view(t, self.Hq, self.D), pos, self.base)
                k = rope_torch((h @ lw["wk"]).view(t, self.Hkv, self.D), pos, self.base)
                v = (h @ lw["wv"]).view(t, self.Hkv, self.D)
                k_pools[l][r, :, :t] = k.permute(1, 0, 2)
                v_pools[l][r, :, :t] = v.permute(1, 0, 2)
                kk = k.repeat_interleave(g, dim=1).permute(1, 0, 2)  # [Hq][t][D]
                vv = v.repeat_interleave(g, dim=1).permute(1, 0, 2)
                s = (q.permute(1, 0, 2) @ kk.transpose(1, 2)) / math.sqrt(self.D)
                ii = torch.arange(t, device=s.device)
                allow = ii[None, :] <= ii[:, None]
                if window > 0:
                    allow &= ii[None, :] >= ii[:, None] - window + 1
                s = s.masked_fill(~allow[None], float("-inf"))
                o = (torch.softmax(s, -1) @ vv).permute(1, 0, 2).reshape(t, -1)
                x = x + o @ lw["wo"]
                x = self._mlp(x, lw)
            out[r, 0] = self._logits(x[t - 1])
        return out

    @torch.no_grad()
    def step(self, st, k_pools, v_pools, fused=False, hook=None):
        """One decode forward of the b_live leaves: context GEMMs around the library's
        trie_rope_kv_append + trie_attn_decode (fused=True: the one-launch
        trie_attn_decode_rope).  hook(layer, q, k, v, o), if given, sees every layer's
        un-rotated projections and the attention output.  Returns logits [R][b_live][V]
        fp32."""
        R, b = st.R, st.b_live
        leaf = st.leaf[:, :b].long()
        tok = torch.gather(st.token.long(), 1, leaf)  # tokens of the pending leaves
        x = self.emb[tok.view(-1)]
        for l, lw in enumerate(self.layers):
            h = rms_norm(x, lw["g1"], self.eps)
            q = (h @ lw["wq"]).view(R, b, self.Hq, self.D).contiguous()
            k = (h @ lw["wk"]).view(R, b, self.Hkv, self.D).contiguous()
            v = (h @ lw["wv"]).view(R, b, self.Hkv, self.D).contiguous()
            o = torch.empty_like(q)
            if fused:
                st.attn_decode_rope(q, k, v, k_pools[l], v_pools[l], self.base, o)
            else:
                st.rope_kv_append(q, k, v, k_pools[l], v_pools[l], self.base)
                st.attn_decode(q, k_pools[l], v_pools[l], o)
            if hook is not None:
                hook(l, q, k, v, o)
            x = x + o.view(R * b, -1) @ lw["wo"]
            x = self._mlp(x, lw)
        return self._logits(x).view(R, b, self.V)


class ShapedModel:
    """Random-init bf16 decoder shaped like Phi-3.5-mini / Llama-3.1-8B / Mistral-Small-24B
    (north_star: "model GEMMs ... random-init MHA, GQA and SWA layers shaped like ...,
    using cuBLAS ... context, not product").  One decode step of the b_live leaves:

        x = E[token of each leaf];  per layer:  h = rmsnorm(x) g1;  q, k, v = h Wq, h Wk, h Wv
        (cuBLAS);  trie_attn_decode_rope (the library: RoPE at trie depth, append, trie
        attention);  x += o Wo;  x += (silu(h2 Wg) * (h2 Wu)) Wd with h2 = rmsnorm(x) g2;
        logits = kappa * (rmsnorm(x) gf) W_lm  (fp32, [R][b_live][V]).

    Weights are N(0, 1 / fan_in) bf16 from a seeded torch generator; every buffer is
    preallocated per b_live so a step is CUDA-graph capturable.  The prompt's K/V rows are
    whatever the caller put in the pools (the bench's synthetic prompt rows)."""

    def __init__(self, L, d, Hq, Hkv, D, ffn, V, rope_base, kappa=3.0, eps=1e-5, seed=0,
                 device="cuda", q_heads=None, kv_heads=None):
        g = torch.Generator(device=device)
        g.manual_seed(0x7472696500 + seed)
        self.L, self.d, self.D, self.ffn, self.V = L, d, D, ffn, V
        # local heads (KV-head shard: this rank's slice); O-proj reads all Hq heads
        self.Hq_all, self.Hq, self.Hkv = Hq, q_heads or Hq, kv_heads or Hkv
        self.base, self.kappa, self.eps = rope_base, kappa, eps

        def W(n_in, n_out):
            return (torch.randn(n_in, n_out, generator=g, device=device, dtype=torch.bfloat16)
                    * (1.0 / math.sqrt(n_in))).to(torch.bfloat16)
        self.layers = []
        for _ in range(L):
            self.layers.append(dict(
                wq=W(d, self.Hq * D), wk=W(d, self.Hkv * D), wv=W(d, self.Hkv * D),
                wo=W(Hq * D, d), wgu=W(d, 2 * ffn), wd=W(ffn, d),
                g1=torch.ones(d, device=device, dtype=torch.bfloat16),
                g2=torch.ones(d, device=device, dtype=torch.bfloat16)))
        self.emb = torch.randn(V, d, generator=g, device=device, dtype=torch.bfloat16)
        self.lm = W(d, V)
        self.gf = torch.ones(d, device=device, dtype=torch.bfloat16)
        self.device = device
        self.bufs = {}

    def weight_bytes(self):
        n = self.emb.numel() + self.lm.numel() + self.gf.numel()
        for lw in self.layers:
            n += sum(t.numel() for t in lw.values())
        return 2 * n

    def _buf(self, R, b):
        key = (R, b)
        if key not in self.bufs:
            M, dev, bf = R * b, self.device, torch.bfloat16
            self.bufs[key] = dict(
                q=torch.empty(R, b, self.Hq, self.D, device=dev, dtype=bf),
                k=torch.empty(R, b, self.Hkv, self.D, device=dev, dtype=bf),
                v=torch.empty(R, b, self.Hkv, self.D, device=dev, dtype=bf),
                o=torch.empty(R, b, self.Hq, self.D, device=dev, dtype=bf),
                logits=torch.empty(R, b, self.V, device=dev, dtype=torch.float32))
        return self.bufs[key]

    def _norm(self, x, g):
        xf = x.float()
        return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.eps)).to(x.dtype) * g

    @torch.no_grad()
    def step(self, st, k_pools, v_pools, gather=None, events=None):
        """One decode step's forward for the handle's b_live leaves; returns the fp32 logits
        buffer [R][b_live][V].  gather(o) -> [R][b][Hq_all][D] (KV-head shard; None: o).
        events: optional list of (start, end) CUDA event pairs, one per layer's attention
        launch, + one for the LM head."""
        R, b = st.R, st.b_live
        B = self._buf(R, b)
        tok = torch.gather(st.token, 1, st.leaf[:, :b].long()).view(-1).long()
        x = self.emb.index_select(0, tok)                      # [R*b][d]
        for l, lw in enumerate(self.layers):
            h = self._norm(x, lw["g1"])
            torch.mm(h, lw["wq"], out=B["q"].view(R * b, -1))
            torch.mm(h, lw["wk"], out=B["k"].view(R * b, -1))
            torch.mm(h, lw["wv"], out=B["v"].view(R * b, -1))
            if events is not None:
                events[l][0].record()
            st.attn_decode_rope(B["q"], B["k"], B["v"], k_pools[l], v_pools[l], self.base, B["o"])
            if events is not None:
                events[l][1].record()
            o = B["o"] if gather is None else gather(B["o"])
            x = x + torch.mm(o.reshape(R * b, -1), lw["wo"])
            h2 = self._norm(x, lw["g2"])
            gu = torch.mm(h2, lw["wgu"])
            x = x + torch.mm(torch.nn.functional.silu(gu[:, : self.ffn]) * gu[:, self.ffn:], lw["wd"])
        if events is not None:
            events[self.L][0].record()
        lg = torch.mm(self._norm(x, self.gf), self.lm)
        B["logits"].view(R * b, -1).copy_(lg)
        B["logits"].mul_(self.kappa)
        if events is not None:
            events[self.L][1].record()
        return B["logits"]
