"""B200-native (sm_100a) hot path of trie-based parallel beam decoding (arXiv 2502.00085).

libtriedecode.so (csrc/, C ABI in include/triedecode.h) holds every step of the hot path:
trie_rope_kv_append, trie_attn_decode, trie_beam_step (+ trie_append), trie_prune_compact.
`_lib` is the ctypes binding (same names), `trie.TrieState` owns one handle's workspace,
`model` is the random-init model context (cuBLAS GEMMs via torch -- context, not product),
`decode` runs the beam loop on one GPU, `dist` partitions requests over ranks.
"""
from . import _lib  # noqa: F401

__all__ = ["_lib"]
