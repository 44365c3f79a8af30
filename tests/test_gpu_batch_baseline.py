"""GPU: the NEXT-2 batch-beam-search baseline.

trie_batch_reorder_kv is batch beam search's cache reorder (Alg. 1 l.6-7): beam r
of a request continues parent beam j, so its generated rows become a copy of j's.  Checked
bit-exactly against a numpy gather; then the baseline's per-beam attention (single-beam
chains) is checked against the trie attention of the same beams (trie == batch, §3.3:
the tree attention of a beam reads exactly its sequence's rows), and the bench arm runs."""
import json
import os
import subprocess
import sys
import zlib

import numpy as np
import pytest
import torch

import synth
from oracle.kernels_ref import build_tries
from tests.gpu_util import need_gpu, per_request_selections, rel_err

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("R,b,Hkv,D,cap,L,dt", [
    (3, 4, 2, 128, 192, 2, torch.bfloat16),
    (2, 8, 8, 96, 320, 3, torch.bfloat16),
    (1, 32, 1, 64, 128, 1, torch.float32),
])
def test_batch_reorder_matches_gather(R, b, Hkv, D, cap, L, dt):
    need_gpu()
    from paper_2502_00085_b200 import _lib
    rng = np.random.default_rng(R * 100 + b)
    shape = (L, R * b, Hkv, cap, D)
    src_k = torch.randn(shape, device="cuda").to(dt)
    src_v = torch.randn(shape, device="cuda").to(dt)
    dst_k = torch.randn(shape, device="cuda").to(dt)
    dst_v = torch.randn(shape, device="cuda").to(dt)
    dk0, dv0 = dst_k.clone(), dst_v.clone()
    par = rng.integers(0, b, (R, b)).astype(np.int32)
    t = np.repeat(rng.integers(1, cap // 2, R), b).astype(np.int32)           # per beam
    n = np.minimum(t + np.repeat(rng.integers(0, cap // 2, R), b), cap).astype(np.int32)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.trie_batch_reorder_kv(R, b, Hkv, D, cap, torch.as_tensor(par, device="cuda"),
                               torch.as_tensor(t, device="cuda"), torch.as_tensor(n, device="cuda"),
                               list(src_k), list(src_v), list(dst_k), list(dst_v), status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    sk, sv = src_k.cpu(), src_v.cpu()
    ek, ev = dk0.cpu(), dv0.cpu()
    for i in range(R):
        for r in range(b):
            d, s_ = i * b + r, i * b + int(par[i, r])
            lo, hi = int(t[d]), int(n[s_])
            ek[:, d, :, lo:hi] = sk[:, s_, :, lo:hi]
            ev[:, d, :, lo:hi] = sv[:, s_, :, lo:hi]
    assert torch.equal(dst_k.cpu(), ek) and torch.equal(dst_v.cpu(), ev)


def test_batch_reorder_rejects_bad_parent_and_in_place():
    need_gpu()
    from paper_2502_00085_b200 import _lib
    R, b, Hkv, D, cap = 1, 2, 1, 64, 64
    p = torch.zeros(1, R * b, Hkv, cap, D, dtype=torch.bfloat16, device="cuda")
    q = torch.zeros_like(p)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    one = torch.ones(R * b, dtype=torch.int32, device="cuda")
    _lib.trie_batch_reorder_kv(R, b, Hkv, D, cap, torch.tensor([[0, 5]], dtype=torch.int32, device="cuda"),
                               one, one * 3, [p[0]], [p[0]], [q[0]], [q[0]], status)
    torch.cuda.synchronize()
    assert int(status.item()) & _lib.TRIE_ST_PARENT
    with pytest.raises(_lib.TrieError):
        _lib.trie_batch_reorder_kv(R, b, Hkv, D, cap, one.view(1, 2), one, one, [p[0]], [p[0]], [p[0]], [q[0]])


def test_batch_chains_attention_equals_trie_attention():
    """The baseline's per-beam attention over private caches == trie attention over the
    shared pool, for the same beams (bf16 tolerance 2e-2, reading R24)."""
    need_gpu()
    from paper_2502_00085_b200.trie import TrieState
    R, b, t, Hq, Hkv, D, V, steps = 2, 4, 150, 8, 2, 128, 300, 9
    seed = zlib.crc32(b"batch-vs-trie") % 1000
    prompts, lens = synth.prompts(seed, R, t, V)
    sels = per_request_selections(seed, R, steps, b, V, 0.5)
    cap = (t + b * steps + b + 63) // 64 * 64
    st = TrieState(R, b, t, cap, 1, Hq, Hkv, D, V, prompts, lens, dtype=torch.bfloat16)
    kp, vp = st.new_pools()
    for par, tok in sels:
        st.append(torch.as_tensor(par, device="cuda"), torch.as_tensor(tok, device="cuda"))
        st.prune_compact(kp, vp)
    tries = build_tries(prompts, lens, sels, b, g=1, final_gc=True)
    K = torch.as_tensor(synth.normal(seed, 1, (R, Hkv, cap, D)), dtype=torch.float32).to(torch.bfloat16).cuda()
    Vv = torch.as_tensor(synth.normal(seed, 2, (R, Hkv, cap, D)), dtype=torch.float32).to(torch.bfloat16).cuda()
    kp[0].copy_(K)
    vp[0].copy_(Vv)
    q = torch.as_tensor(synth.normal(seed, 3, (R, b, Hq, D)), dtype=torch.float32).to(torch.bfloat16).cuda()
    out_trie = torch.empty_like(q)
    st.attn_decode(q, kp[0], vp[0], out_trie, rows_hint=t + steps)
    # private caches: beam j's sequence rows in order (a chain of t + steps nodes)
    n_seq = t + steps
    ccap = (n_seq + 63) // 64 * 64
    ch = TrieState(R * b, 1, n_seq, ccap, 1, Hq, Hkv, D, V, np.zeros((R * b, n_seq), np.int32),
                   [n_seq] * (R * b), dtype=torch.bfloat16)
    ck, cv = ch.new_pools()
    for i in range(R):
        T = tries[i]
        for j, leaf in enumerate(T.leaves):
            path, n = [], leaf
            while n >= 0:
                path.append(n)
                n = T.parent[n]
            path = path[::-1]
            assert len(path) == n_seq
            ck[0, i * b + j, :, :n_seq] = K[i][:, path]
            cv[0, i * b + j, :, :n_seq] = Vv[i][:, path]
    out_batch = torch.empty(R * b, 1, Hq, D, dtype=torch.bfloat16, device="cuda")
    ch.attn_decode(q.view(R * b, 1, Hq, D), ck[0], cv[0], out_batch, rows_hint=n_seq)
    torch.cuda.synchronize()
    assert rel_err(out_batch.view(R, b, Hq, D).float().cpu().numpy(),
                   out_trie.float().cpu().numpy()) <= 2e-2


def test_bench_batch_arm_runs():
    need_gpu()
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "batch", "--workload",
                          "llama", "--requests", "4", "--steps", "8", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["impl"] == "batch" and res["value"] > 0 and res["gpu_launches"] > 0


def test_bench_two_ranks_request_dp():
    """bench.py's N > 1 path (request data parallel, one process per rank, max-over-ranks
    timing) on one GPU: two ranks share cuda:0 through the gloo test mode."""
    need_gpu()
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--workload", "llama", "--requests", "4", "--steps", "6", "--warmup", "3",
                          "--no-cpu-baseline", "--no-e2e"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads([l for l in out.stdout.strip().splitlines() if l.startswith("{")][-1])
    assert res["n_gpus"] == 2 and res["value"] > 0 and res["scaling"] == "weak"
    assert res["config"]["parallelism"] == "request-dp2"


@pytest.mark.parametrize("seed,Hkv,b,R,use_eos", [(0, 4, 3, 2, False), (7, 1, 8, 2, False), (3, 2, 4, 3, False),
                                                   (0, 4, 3, 2, True), (2, 4, 5, 2, True)])
def test_gpu_batch_beam_search_equals_gpu_trie_decode(seed, Hkv, b, R, use_eos):
    """The paper's equivalence on the GPU, end to end on the tiny decoder
    (fp32): batch beam search (Alg. 1) built from the library's calls -- private
    single-beam caches per beam, trie_beam_step for the top-b, trie_batch_reorder_kv for
    the cache reorder -- selects exactly what the trie decode selects at every step."""
    need_gpu()
    from paper_2502_00085_b200 import _lib
    from paper_2502_00085_b200.decode import trie_beam_decode
    from paper_2502_00085_b200.model import TinyModel
    from paper_2502_00085_b200.trie import TrieState
    t, s, V, D = 8, 12, 256, 16
    prompts, lens = synth.prompts(seed, R, t, V)
    gm = TinyModel(seed, Hkv=Hkv)
    st = TrieState(R, b, t, t + b * s + b, 2, 4, Hkv, D, V, prompts, lens, dtype=torch.float32)
    kp, vp = st.new_pools()
    eos = None
    if use_eos:  # NEXT-3: an EOS id the trie decode selects at step 3 (absorbing, R5b)
        _, _, _, tr0 = trie_beam_decode(gm, st, kp, vp, prompts, lens, 3, g=1, record=True)
        eos = int(tr0[2]["tok"][0, 0])
        st.reset()
    _, _, _, trace = trie_beam_decode(gm, st, kp, vp, prompts, lens, s, g=1, record=True, eos=eos)
    # batch beam search: R*b single-beam chains (prompt replicated), two pool sets
    rep = np.repeat(prompts, b, axis=0)
    rlen = np.repeat(lens, b)
    ccap = t + s + 1
    ch = TrieState(R * b, 1, t, ccap, 2, 4, Hkv, D, V, rep, rlen, dtype=torch.float32)
    sel = TrieState(R, b, t, t + b * s + b, 0, 4, Hkv, D, V, prompts, lens, dtype=torch.float32)
    sel.set_eos(-1 if eos is None else eos)
    P = [ch.new_pools(), ch.new_pools()]
    logits = gm.prefill(rep, rlen, P[0][0], P[0][1])
    P[1][0].copy_(P[0][0])
    P[1][1].copy_(P[0][1])
    zeros = torch.zeros(R * b, dtype=torch.int32, device="cuda")
    cur = 0
    for k in range(1, s + 1):
        lg = logits.view(R, b, V)
        if k == 1:
            lg = lg[:, :1].contiguous()  # one live beam: the prompt
        sp = torch.empty(R, b, dtype=torch.int32, device="cuda")
        tk = torch.empty_like(sp)
        sc = torch.empty(R, b, dtype=torch.float32, device="cuda")
        sel.beam_step(lg, sp, tk, sc)
        _lib.trie_batch_reorder_kv(R, b, Hkv, D, ccap, sp, ch.prompt_len, ch.n_nodes,
                                   list(P[cur][0]), list(P[cur][1]), list(P[1 - cur][0]), list(P[1 - cur][1]))
        ch.append(zeros, tk.view(-1))
        cur = 1 - cur
        assert sp.cpu().numpy().tolist() == trace[k - 1]["par"].tolist(), f"step {k}: parents differ"
        assert tk.cpu().numpy().tolist() == trace[k - 1]["tok"].tolist(), f"step {k}: tokens differ"
        np.testing.assert_allclose(sc.cpu().numpy(), trace[k - 1]["score"], rtol=1e-4, atol=1e-4)
        if k < s:
            logits = gm.step(ch, P[cur][0], P[cur][1])
    assert ch.status() == 0 and sel.status() == 0
