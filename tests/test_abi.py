"""CPU-side checks of the boundary: the C-ABI library builds for sm_100a, loads, and exports
every symbol include/triedecode.h declares; the binding exposes the same names; no compute
call is made (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "triedecode.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(trie_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2502_00085_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_four_named_calls():
    names = _declared()
    for n in ("trie_create", "trie_attn_decode", "trie_beam_step", "trie_prune_compact"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_names_match_header():
    from paper_2502_00085_b200 import _lib
    assert sorted(_lib.SYMBOLS) == _declared()
    for n in _declared():
        assert callable(getattr(_lib, n))


def test_library_is_sm100a(lib):
    path = os.path.join(ROOT, "paper_2502_00085_b200", "libtriedecode.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_string(lib):
    from paper_2502_00085_b200 import _lib
    assert _lib.trie_version() >> 16 == 1
    assert isinstance(_lib.load().trie_last_error(), bytes)


def test_validation_without_gpu(lib):
    """Argument validation runs on the host: bad shapes are rejected before any launch."""
    from paper_2502_00085_b200 import _lib
    bad = [
        _lib.make_cfg(1, 33, 8, 100, 1, 4, 4, 16, 256),     # b > 32
        _lib.make_cfg(1, 4, 8, 100, 1, 6, 4, 16, 256),      # Hq % Hkv != 0
        _lib.make_cfg(1, 4, 8, 100, 1, 4, 4, 24, 256),      # D % 16 != 0
        _lib.make_cfg(1, 8, 8, 100, 1, 4, 4, 16, 4),        # b > V
        _lib.make_cfg(1, 4, 8, 9, 1, 4, 4, 16, 256),        # capacity < t + b
    ]
    for c in bad:
        with pytest.raises(_lib.TrieError):
            _lib.trie_workspace_bytes(c)
    ok = _lib.make_cfg(2, 4, 8, 100, 2, 4, 4, 16, 256)
    assert _lib.trie_workspace_bytes(ok) > 0
