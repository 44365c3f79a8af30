"""TrieState: owns the workspace of one trie handle and exposes the C ABI calls as methods.

PyTorch only allocates device memory and provides the stream; every operation on the
trie, the KV pools and the logits runs in libtriedecode's kernels (argument marshalling
only here).
"""
from __future__ import annotations

import torch

from . import _lib as L


class TrieState:
    def __init__(self, R, b, t_max, capacity, n_layers, Hq, Hkv, D, V, prompt_tokens, prompt_lens,
                 window=0, gc_interval=1, dtype=torch.bfloat16, device="cuda", stream=None, n_pages=0):
        if not torch.cuda.is_available():
            raise L.TrieError("no CUDA device: libtriedecode has no CPU path")
        self.kv_dtype = L.TRIE_BF16 if dtype == torch.bfloat16 else L.TRIE_F32
        self.dtype = dtype
        self.cfg = L.make_cfg(R, b, t_max, capacity, n_layers, Hq, Hkv, D, V, window, gc_interval,
                              self.kv_dtype, n_pages)
        self.n_pages = n_pages
        self.R, self.b, self.t_max, self.cap = R, b, t_max, capacity
        self.L, self.Hq, self.Hkv, self.D, self.V, self.window = n_layers, Hq, Hkv, D, V, window
        self.device = device
        nbytes = L.trie_workspace_bytes(self.cfg)
        self.ws = torch.zeros(nbytes + 256, dtype=torch.uint8, device=device)
        off = (-self.ws.data_ptr()) % 256
        self.ws_al = self.ws[off: off + nbytes]
        toks = torch.as_tensor(prompt_tokens, dtype=torch.int32).reshape(R, t_max).to(device)
        self.h = L.trie_create(self.cfg, self.ws_al, list(prompt_lens), toks, stream)
        self._toks = toks
        self._views()
        self.attn_scratch = None
        self.hyp_scratch = None

    def _views(self):
        a = L.trie_get_arrays(self.h)
        base = self.ws_al.data_ptr()

        def view(ptr, n, dt, shape):
            o = ptr - base
            return self.ws_al[o: o + n * 4].view(dt).view(*shape)
        R, cap = self.R, self.cap
        self.token = view(a.token, R * cap, torch.int32, (R, cap))
        self.parent = view(a.parent, R * cap, torch.int32, (R, cap))
        self.depth = view(a.depth, R * cap, torch.int32, (R, cap))
        self.beam_mask = view(a.beam_mask, R * cap, torch.int32, (R, cap))  # uint32 bits
        self.leaf = view(a.leaf, R * 32, torch.int32, (R, 32))
        self.score = view(a.score, R * 32, torch.float32, (R, 32))
        self.n_nodes = view(a.n_nodes, R, torch.int32, (R,))
        self.prompt_len = view(a.prompt_len, R, torch.int32, (R,))
        self.finished = view(a.finished, R * 32, torch.int32, (R, 32))  # uint32 flags
        self.status_word = view(a.status, 1, torch.int32, (1,))         # TRIE_ST_* bits
        self.page_table = (view(a.page_table, R * (cap // 64), torch.int32, (R, cap // 64))
                           if self.n_pages else None)                   # NEXT-2 paged pools

    @property
    def b_live(self) -> int:
        return L.trie_get_arrays(self.h).b_live

    @property
    def steps(self) -> int:
        return L.trie_get_arrays(self.h).steps

    def new_pools(self):
        """Zero-initialised K and V pools, one tensor per layer: dense [R][Hkv][cap][D], or
        paged [n_pages][Hkv][64][D] (include/triedecode.h "KV pool layouts")."""
        shape = ((self.L, self.n_pages, self.Hkv, 64, self.D) if self.n_pages
                 else (self.L, self.R, self.Hkv, self.cap, self.D))
        return (torch.zeros(shape, dtype=self.dtype, device=self.device),
                torch.zeros(shape, dtype=self.dtype, device=self.device))

    # ---- paged pools (NEXT-2): host-side views for prefill and tests (plain indexing) ----
    def prompt_pages(self, r):
        """Fixed pages of request r's prompt (off_r .. off_r + ceil(t_r / 64) - 1)."""
        lens = self.prompt_len.cpu().tolist()
        off = sum((int(t) + 63) // 64 for t in lens[:r])
        return list(range(off, off + (int(lens[r]) + 63) // 64))

    def write_rows(self, pool_l, rows):
        """Write dense rows [R][Hkv][n][D] (slots 0..n-1 of every request) into a layer's
        pool, through the page table when paged (the caller's prefill)."""
        n = rows.shape[2]
        if not self.n_pages:
            pool_l[:, :, :n] = rows
            return
        pt = self.page_table.cpu()
        for r in range(self.R):
            for blk in range((n + 63) // 64):
                if int(pt[r, blk]) < 0:  # block not mapped (beyond the request's N)
                    continue
                m = min(64, n - blk * 64)
                pool_l[int(pt[r, blk]), :, :m] = rows[r, :, blk * 64: blk * 64 + m]

    def dense_view(self, pool_l, n=None, requests=None):
        """[R][Hkv][n][D] copy of a layer's pool in slot order (tests); `requests`: only those
        (in that order)."""
        n = self.cap if n is None else n
        reqs = list(range(self.R)) if requests is None else list(requests)
        if not self.n_pages:
            return pool_l[reqs, :, :n].clone()
        pt = self.page_table.cpu()
        out = torch.zeros(len(reqs), self.Hkv, n, self.D, dtype=pool_l.dtype, device=pool_l.device)
        for i, r in enumerate(reqs):
            for blk in range((n + 63) // 64):
                pg = int(pt[r, blk])
                if pg < 0:
                    continue
                m = min(64, n - blk * 64)
                out[i, :, blk * 64: blk * 64 + m] = pool_l[pg, :, :m]
        return out

    def swa_evict(self, stream=None):
        """NEXT-3: free the pages of prompt blocks below every live beam's window."""
        L.trie_swa_evict(self.h, stream)

    def page_stats(self, stream=None) -> dict:
        return L.trie_page_stats(self.h, stream)

    # ---- C ABI calls ----------------------------------------------------------------
    def set_eos(self, eos_id: int):
        """NEXT-3: EOS as an absorbing token (trie_set_eos); -1 disables."""
        L.trie_set_eos(self.h, eos_id)

    def reset(self, stream=None):
        L.trie_reset(self.h, stream)

    def rope_kv_append(self, q, k_new, v_new, k_pool_l, v_pool_l, rope_theta, stream=None):
        L.trie_rope_kv_append(self.h, q, k_new, v_new, k_pool_l, v_pool_l, rope_theta, stream)

    def attn_decode(self, q, k_pool_l, v_pool_l, out, lse=None, rows_hint=0, use_mask=True,
                    stream=None):
        b_live = self.b_live
        need = L.trie_attn_scratch_bytes(self.cfg, b_live, rows_hint)
        if self.attn_scratch is None or self.attn_scratch.numel() < need:
            # zero-initialised once (counters in the scratch are left at zero by every launch)
            self.attn_scratch = torch.zeros(need, dtype=torch.uint8, device=self.device)
        L.trie_attn_decode(self.cfg, b_live, q, k_pool_l, v_pool_l, self.prompt_len, self.parent,
                           self.depth, self.leaf, self.n_nodes, self.beam_mask if use_mask else None,
                           self.window, rows_hint, out, lse, self.attn_scratch, stream,
                           status=self.status_word)

    def attn_decode_rope(self, q, k_new, v_new, k_pool_l, v_pool_l, rope_theta, out, lse=None,
                         rows_hint=0, stream=None):
        """Fused a-1 + a-3: RoPE at depth + KV append + trie attention in one launch."""
        need = L.trie_attn_scratch_bytes(self.cfg, self.b_live, rows_hint)
        if self.attn_scratch is None or self.attn_scratch.numel() < need:
            self.attn_scratch = torch.zeros(need, dtype=torch.uint8, device=self.device)
        L.trie_attn_decode_rope(self.h, q, k_new, v_new, k_pool_l, v_pool_l, rope_theta, rows_hint, out,
                                lse, self.attn_scratch, stream)

    def beam_step(self, logits, sel_parent=None, sel_token=None, new_score=None, stream=None):
        L.trie_beam_step(self.h, logits, sel_parent, sel_token, new_score, stream)

    def append(self, sel_parent, sel_token, new_score=None, stream=None):
        L.trie_append(self.h, sel_parent, sel_token, new_score, stream)

    def prune_compact(self, k_pools, v_pools, stream=None):
        L.trie_prune_compact(self.h, [k_pools[l] for l in range(self.L)],
                             [v_pools[l] for l in range(self.L)], stream)

    def read_hyps(self, max_len, stream=None):
        need = self.R * 32 * (max_len + 1) * 4
        if self.hyp_scratch is None or self.hyp_scratch.numel() < need:
            self.hyp_scratch = torch.empty(need, dtype=torch.uint8, device=self.device)
        return L.trie_read_hyps(self.h, self.R, self.b_live, max_len, self.hyp_scratch, stream)

    def status(self, stream=None) -> int:
        return L.trie_status(self.h, stream)

    def close(self):
        if self.h is not None:
            L.trie_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
