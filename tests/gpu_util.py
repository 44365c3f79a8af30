"""Helpers shared by the -m gpu parity tests (inputs only; no method arithmetic)."""
import numpy as np
import pytest
import torch

import synth


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_00085_b200 import _lib
    _lib.load()  # raises if the library is missing: there is no fallback


def per_request_selections(seed, R, steps, b, V, rho):
    """sel_seq[k] = (parent[R][b], token[R][b]) with an independent dial per request."""
    per = [synth.selections(seed * 1000 + r, steps, b, V, rho) for r in range(R)]
    return [(np.stack([per[r][k][0] for r in range(R)]), np.stack([per[r][k][1] for r in range(R)]))
            for k in range(steps)]


def rel_err(a, ref):
    """Reading R24: per row max|a - ref| / max(max|ref|, 1e-6), rows = leading dims."""
    a = np.asarray(a, np.float64).reshape(-1, np.shape(a)[-1])
    ref = np.asarray(ref, np.float64).reshape(-1, np.shape(ref)[-1])
    den = np.maximum(np.abs(ref).max(axis=1), 1e-6)
    return (np.abs(a - ref).max(axis=1) / den).max()
