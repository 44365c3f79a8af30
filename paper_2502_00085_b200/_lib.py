"""ctypes binding of libtriedecode.so -- argument marshalling only.

The functions below have the C ABI's names (include/triedecode.h) and take torch CUDA
tensors for device pointers; every step of the hot path runs in the library's kernels.
There is no CPU fallback: if the shared library is missing or no CUDA device is present,
the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# TRIE_LIB: an alternative build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("TRIE_LIB") or os.path.join(_HERE, "libtriedecode.so")

TRIE_F32, TRIE_BF16 = 0, 1
TRIE_ST_CAPACITY, TRIE_ST_PARENT, TRIE_ST_EMPTY_ROW, TRIE_ST_LEAF = 1, 2, 4, 8

SYMBOLS = ["trie_workspace_bytes", "trie_create", "trie_reset", "trie_destroy", "trie_get_arrays",
           "trie_rope_kv_append", "trie_attn_scratch_bytes", "trie_attn_decode", "trie_beam_step",
           "trie_append", "trie_prune_compact", "trie_read_hyps", "trie_status", "trie_last_error",
           "trie_version", "trie_launch_count", "trie_attn_decode_rope", "trie_attn_plan_info",
           "trie_batch_reorder_kv", "trie_set_eos", "trie_gather_setup", "trie_gather_wait",
           "trie_ipc_alloc", "trie_ipc_open", "trie_ipc_close", "trie_ipc_free", "trie_page_stats",
           "trie_swa_evict"]


class trie_cfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "n_requests", "beam_width", "max_prompt_len", "capacity", "n_layers", "n_q_heads",
        "n_kv_heads", "head_dim", "vocab", "window", "gc_interval", "kv_dtype", "n_pages")]


class trie_arrays(ctypes.Structure):
    _fields_ = [("token", ctypes.c_void_p), ("parent", ctypes.c_void_p), ("depth", ctypes.c_void_p),
                ("beam_mask", ctypes.c_void_p), ("leaf", ctypes.c_void_p), ("score", ctypes.c_void_p),
                ("n_nodes", ctypes.c_void_p), ("prompt_len", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("b_live", ctypes.c_int32), ("steps", ctypes.c_int32),
                ("finished", ctypes.c_void_p), ("page_table", ctypes.c_void_p), ("page_ctr", ctypes.c_void_p)]


_lib = None


def load(path: str = LIB_PATH):
    """Load the shared library (raises if it is missing -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run `python -m paper_2502_00085_b200.build`")
    lib = ctypes.CDLL(path)
    P, I32, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
    CP = ctypes.POINTER(trie_cfg)
    sig = {
        "trie_workspace_bytes": (ctypes.c_int, [CP, ctypes.POINTER(SZ)]),
        "trie_create": (ctypes.c_int, [CP, P, SZ, P, P, ctypes.POINTER(P), P]),
        "trie_reset": (ctypes.c_int, [P, P]),
        "trie_destroy": (ctypes.c_int, [P]),
        "trie_get_arrays": (ctypes.c_int, [P, ctypes.POINTER(trie_arrays)]),
        "trie_rope_kv_append": (ctypes.c_int, [P, P, P, P, P, P, ctypes.c_float, P]),
        "trie_attn_scratch_bytes": (SZ, [CP, I32, I32]),
        "trie_attn_decode": (ctypes.c_int, [CP, I32, P, P, P, P, P, P, P, P, P, I32, I32, P, P, P,
                                            SZ, P, P]),
        "trie_attn_decode_rope": (ctypes.c_int, [P, P, P, P, P, P, ctypes.c_float, I32, P, P, P, SZ, P]),
        "trie_attn_plan_info": (ctypes.c_int, [CP, I32, I32, P]),
        "trie_beam_step": (ctypes.c_int, [P, P, P, P, P, P]),
        "trie_append": (ctypes.c_int, [P, P, P, P, P]),
        "trie_prune_compact": (ctypes.c_int, [P, P, P, P]),
        "trie_read_hyps": (ctypes.c_int, [P, I32, P, P, P, P, SZ, P]),
        "trie_status": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_uint32), P]),
        "trie_last_error": (ctypes.c_char_p, []),
        "trie_version": (ctypes.c_int, []),
        "trie_launch_count": (ctypes.c_ulonglong, []),
        "trie_batch_reorder_kv": (ctypes.c_int, [I32] * 7 + [P] * 3 + [P] * 4 + [P, P]),
        "trie_set_eos": (ctypes.c_int, [P, I32]),
        "trie_page_stats": (ctypes.c_int, [P, P, P]),
        "trie_swa_evict": (ctypes.c_int, [P, P]),
        "trie_gather_setup": (ctypes.c_int, [P, I32, I32, P, P]),
        "trie_gather_wait": (ctypes.c_int, [P, P, P]),
        "trie_ipc_alloc": (ctypes.c_int, [SZ, ctypes.POINTER(P), P]),
        "trie_ipc_open": (ctypes.c_int, [P, ctypes.POINTER(P)]),
        "trie_ipc_close": (ctypes.c_int, [P]),
        "trie_ipc_free": (ctypes.c_int, [P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class TrieError(RuntimeError):
    pass


def _check(rc: int, what: str):
    if rc != 0:
        raise TrieError(f"{what} failed ({rc}): {load().trie_last_error().decode()}")


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if not t.is_cuda:
        raise TrieError("expected a CUDA tensor (no CPU path)")
    return t.data_ptr()


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def make_cfg(R, b, t_max, capacity, L, Hq, Hkv, D, V, window=0, gc_interval=1, kv_dtype=TRIE_BF16,
             n_pages=0):
    return trie_cfg(R, b, t_max, capacity, L, Hq, Hkv, D, V, window, gc_interval, kv_dtype, n_pages)


# ---- entry points (same names as the C ABI) ------------------------------------------
def trie_workspace_bytes(cfg: trie_cfg) -> int:
    n = ctypes.c_size_t(0)
    _check(load().trie_workspace_bytes(ctypes.byref(cfg), ctypes.byref(n)), "trie_workspace_bytes")
    return n.value


def trie_create(cfg: trie_cfg, workspace, prompt_lens, prompt_tokens, stream=None):
    lens = (ctypes.c_int32 * cfg.n_requests)(*[int(x) for x in prompt_lens])
    h = ctypes.c_void_p()
    _check(load().trie_create(ctypes.byref(cfg), _ptr(workspace), workspace.numel() * workspace.element_size(),
                              ctypes.cast(lens, ctypes.c_void_p), _ptr(prompt_tokens), ctypes.byref(h),
                              _stream(stream)), "trie_create")
    return h


def trie_reset(h, stream=None):
    _check(load().trie_reset(h, _stream(stream)), "trie_reset")


def trie_destroy(h):
    _check(load().trie_destroy(h), "trie_destroy")


def trie_get_arrays(h) -> trie_arrays:
    a = trie_arrays()
    _check(load().trie_get_arrays(h, ctypes.byref(a)), "trie_get_arrays")
    return a


def trie_rope_kv_append(h, q, k_new, v_new, k_pool, v_pool, rope_theta: float, stream=None):
    _check(load().trie_rope_kv_append(h, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(k_pool), _ptr(v_pool),
                                      float(rope_theta), _stream(stream)), "trie_rope_kv_append")


def trie_attn_scratch_bytes(cfg: trie_cfg, b_live: int, rows_hint: int = 0) -> int:
    return int(load().trie_attn_scratch_bytes(ctypes.byref(cfg), b_live, rows_hint))


def trie_attn_decode(cfg, b_live, q, k_pool, v_pool, prompt_len, parent, depth, leaf_ids, n_nodes,
                     beam_mask, window, rows_hint, out, lse, scratch, stream=None, status=None):
    sb = 0 if scratch is None else scratch.numel() * scratch.element_size()
    _check(load().trie_attn_decode(ctypes.byref(cfg), b_live, _ptr(q), _ptr(k_pool), _ptr(v_pool),
                                   _ptr(prompt_len), _ptr(parent), _ptr(depth), _ptr(leaf_ids),
                                   _ptr(n_nodes), _ptr(beam_mask), window, rows_hint, _ptr(out),
                                   _ptr(lse), _ptr(scratch), sb, _ptr(status), _stream(stream)),
           "trie_attn_decode")


def trie_attn_decode_rope(h, q, k_new, v_new, k_pool, v_pool, rope_theta, rows_hint, out, lse, scratch,
                          stream=None):
    sb = 0 if scratch is None else scratch.numel() * scratch.element_size()
    _check(load().trie_attn_decode_rope(h, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(k_pool), _ptr(v_pool),
                                        float(rope_theta), rows_hint, _ptr(out), _ptr(lse), _ptr(scratch), sb,
                                        _stream(stream)), "trie_attn_decode_rope")


def trie_beam_step(h, logits, sel_parent_beam=None, sel_token=None, new_score=None, stream=None):
    _check(load().trie_beam_step(h, _ptr(logits), _ptr(sel_parent_beam), _ptr(sel_token),
                                 _ptr(new_score), _stream(stream)), "trie_beam_step")


def trie_append(h, sel_parent_beam, sel_token, new_score=None, stream=None):
    _check(load().trie_append(h, _ptr(sel_parent_beam), _ptr(sel_token), _ptr(new_score),
                              _stream(stream)), "trie_append")


def trie_prune_compact(h, k_pools, v_pools, stream=None):
    L = len(k_pools)
    kp = (ctypes.c_void_p * max(L, 1))(*[_ptr(x) for x in k_pools])
    vp = (ctypes.c_void_p * max(L, 1))(*[_ptr(x) for x in v_pools])
    _check(load().trie_prune_compact(h, ctypes.cast(kp, ctypes.c_void_p), ctypes.cast(vp, ctypes.c_void_p),
                                     _stream(stream)), "trie_prune_compact")


def trie_set_eos(h, eos_id: int):
    _check(load().trie_set_eos(h, eos_id), "trie_set_eos")


def trie_batch_reorder_kv(R, b, Hkv, D, cap, sel_parent_beam, prompt_len, n_rows, src_k, src_v,
                          dst_k, dst_v, status=None, stream=None):
    """NEXT-2 baseline: batch beam search's per-beam cache reorder (see the header).
    src_*/dst_*: sequences of per-layer [R*b][Hkv][cap][D] pools."""
    L = len(src_k)
    arr = [(ctypes.c_void_p * L)(*[_ptr(x) for x in pools]) for pools in (src_k, src_v, dst_k, dst_v)]
    esz = src_k[0].element_size()
    _check(load().trie_batch_reorder_kv(R, b, L, Hkv, D, cap, esz, _ptr(sel_parent_beam), _ptr(prompt_len),
                                        _ptr(n_rows), *arr, _ptr(status), _stream(stream)),
           "trie_batch_reorder_kv")


def trie_read_hyps(h, R: int, b_live: int, max_len: int, scratch, stream=None):
    import numpy as np
    toks = np.zeros((R, b_live, max_len), np.int32)
    lens = np.zeros((R, b_live), np.int32)
    scores = np.zeros((R, b_live), np.float32)
    _check(load().trie_read_hyps(h, max_len, toks.ctypes.data, lens.ctypes.data, scores.ctypes.data,
                                 _ptr(scratch), scratch.numel() * scratch.element_size(), _stream(stream)),
           "trie_read_hyps")
    return toks, lens, scores


def trie_status(h, stream=None) -> int:
    bits = ctypes.c_uint32(0)
    _check(load().trie_status(h, ctypes.byref(bits), _stream(stream)), "trie_status")
    return bits.value


def trie_version() -> int:
    return load().trie_version()


def trie_last_error() -> str:
    return load().trie_last_error().decode()


def trie_launch_count() -> int:
    return int(load().trie_launch_count())


ATTN_PATHS = {0: "cuda-core", 1: "narrow-mma.sync", 2: "wide-mma.sync", 3: "tcgen05-tmem"}


def trie_attn_plan_info(cfg: trie_cfg, b_live: int, rows_hint: int = 0) -> dict:
    info = (ctypes.c_int32 * 4)()
    _check(load().trie_attn_plan_info(ctypes.byref(cfg), b_live, rows_hint, ctypes.cast(info, ctypes.c_void_p)),
           "trie_attn_plan_info")
    return dict(path=ATTN_PATHS.get(info[0], str(info[0])), splits=info[1], fused_rope=bool(info[2]), Qg=info[3])


# ---- NEXT-4: fused KV-head-shard all-gather (trie_gather_setup) ---------------------------
def trie_gather_setup(h, world: int, rank: int, peer_out, peer_flags):
    """peer_out / peer_flags: sequences of `world` device pointers (ints) or CUDA tensors --
    every rank's gather buffer and flag array as mapped in this process."""
    outs = (ctypes.c_void_p * max(world, 1))(*[_ptr(x) for x in peer_out])
    flags = (ctypes.c_void_p * max(world, 1))(*[_ptr(x) for x in peer_flags])
    _check(load().trie_gather_setup(h, world, rank, ctypes.cast(outs, ctypes.c_void_p),
                                    ctypes.cast(flags, ctypes.c_void_p)), "trie_gather_setup")


def trie_gather_wait(h, gathered_out=None, stream=None):
    _check(load().trie_gather_wait(h, _ptr(gathered_out), _stream(stream)), "trie_gather_wait")


def trie_ipc_alloc(nbytes: int):
    """cudaMalloc'd, zeroed, IPC-exportable device memory: (device pointer, 64-byte handle)."""
    ptr = ctypes.c_void_p()
    hd = ctypes.create_string_buffer(64)
    _check(load().trie_ipc_alloc(nbytes, ctypes.byref(ptr), ctypes.cast(hd, ctypes.c_void_p)), "trie_ipc_alloc")
    return int(ptr.value), bytes(hd.raw)


def trie_ipc_open(handle: bytes) -> int:
    ptr = ctypes.c_void_p()
    hd = ctypes.create_string_buffer(handle, 64)
    _check(load().trie_ipc_open(ctypes.cast(hd, ctypes.c_void_p), ctypes.byref(ptr)), "trie_ipc_open")
    return int(ptr.value)


def trie_ipc_close(ptr: int):
    _check(load().trie_ipc_close(ptr), "trie_ipc_close")


def trie_ipc_free(ptr: int):
    _check(load().trie_ipc_free(ptr), "trie_ipc_free")


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (the IPC buffers) for torch."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = dict(shape=tuple(shape), typestr=typestr, data=(int(ptr), False),
                                             version=3, strides=None)


def device_tensor(ptr: int, shape, dtype):
    """A torch tensor aliasing device memory at ptr (no copy; the memory stays owned by the
    library's trie_ipc_* calls)."""
    ts = {torch.bfloat16: "<i2", torch.int32: "<i4", torch.float32: "<f4"}[dtype]
    t = torch.as_tensor(_CudaArray(ptr, shape, ts), device="cuda")
    return t.view(dtype) if dtype == torch.bfloat16 else t


# ---- NEXT-2: paged pools -----------------------------------------------------------------
def trie_page_stats(h, stream=None) -> dict:
    st = (ctypes.c_int32 * 3)()
    _check(load().trie_page_stats(h, ctypes.cast(st, ctypes.c_void_p), _stream(stream)), "trie_page_stats")
    return dict(in_use=int(st[0]), peak=int(st[1]), n_pages=int(st[2]))


def trie_swa_evict(h, stream=None):
    _check(load().trie_swa_evict(h, _stream(stream)), "trie_swa_evict")
