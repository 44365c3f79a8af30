"""KV-head sharding (BASELINE.json configs[3]) at world size 2 on ONE GPU:
two processes share cuda:0 over gloo (the driver's runs use NCCL, one rank per GPU).

Each rank holds the SAME requests and trie metadata but only its block of KV heads (and
their query heads); per layer it runs the fused RoPE + append + trie attention
(trie_attn_decode_rope) on its heads and the outputs are all-gathered (dist.gather_heads,
through host memory under gloo).  Checked, step by step in lockstep with the oracle:

* the gathered all-head attention == attn_ref over ALL heads (§3.3) with q / k
  rotated in fp64 at the leaf depth (§3.4) over the oracle trie's rows, <= 2e-2 per row;
* every rank's selection == beam_step_ref on the shared logits (near-tie protocol), and
  the trie metadata (N, token, parent, depth, beam bitsets, leaves) is bit-identical on
  both ranks after every step (identical logits -> identical choices, P:309 multi-GPU);
* bench.py's --workload mistral-shard runs at N = 2 (eager gloo test mode).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import synth
from tests.gpu_util import need_gpu, rel_err

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CFG = dict(R=2, b=4, t=200, Hq=8, Hkv=2, D=128, W=100, L=2, V=300, s=8, base=1e6, seed=77)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bf(x):
    return torch.as_tensor(x, dtype=torch.float32).to(torch.bfloat16)


def _inputs(c, k, l, bl):
    """Seeded all-head inputs of step k, layer l (bf16 values) -- the same on every rank."""
    R, Hq, Hkv, D, seed = c["R"], c["Hq"], c["Hkv"], c["D"], c["seed"]
    st = 1000 + 8 * (k * c["L"] + l)
    return (_bf(synth.normal(seed, st + 1, (R, bl, Hq, D))), _bf(synth.normal(seed, st + 2, (R, bl, Hkv, D))),
            _bf(synth.normal(seed, st + 3, (R, bl, Hkv, D))))


def _rank(rank, world, port, c, q, fused=False):
    import torch.distributed as dist

    from paper_2502_00085_b200.dist import FusedGather, gather_heads, heads_view, kv_head_shard
    from paper_2502_00085_b200.trie import TrieState
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    R, b, t, Hq, Hkv, D, W, L, V, s = (c[k] for k in ("R", "b", "t", "Hq", "Hkv", "D", "W", "L", "V", "s"))
    kv0, nkv, q0, nq = kv_head_shard(Hq, Hkv, world, rank)
    prompts, lens = synth.prompts(c["seed"], R, t, V)
    cap = (t + b * s + b + 63) // 64 * 64
    st = TrieState(R, b, t, cap, L, nq, nkv, D, V, prompts, lens, window=W, dtype=torch.bfloat16)
    kp, vp = st.new_pools()
    fg = FusedGather(st, world, rank) if fused else None
    for l in range(L):
        kp[l][:, :, :t] = _bf(synth.normal(c["seed"], 10 + 2 * l, (R, Hkv, t, D)))[:, kv0:kv0 + nkv].cuda()
        vp[l][:, :, :t] = _bf(synth.normal(c["seed"], 11 + 2 * l, (R, Hkv, t, D)))[:, kv0:kv0 + nkv].cuda()
    rec = []
    for k in range(s):
        bl = 1 if k == 0 else b
        outs = []
        for l in range(L):
            qf, kf, vf = _inputs(c, k, l, bl)
            out = torch.empty(R, bl, nq, D, dtype=torch.bfloat16, device="cuda")
            st.attn_decode_rope(qf[:, :, q0:q0 + nq].contiguous().cuda(), kf[:, :, kv0:kv0 + nkv].contiguous().cuda(),
                                vf[:, :, kv0:kv0 + nkv].contiguous().cuda(), kp[l], vp[l], c["base"], out)
            if fg is not None:  # NEXT-4: stored by the kernel into every rank's buffer
                full = torch.empty(R, bl, Hq, D, dtype=torch.bfloat16, device="cuda")
                fg.wait(full)
                outs.append(full.float().cpu().numpy())
            else:
                outs.append(heads_view(gather_heads(out.cpu())).float().numpy())
        lg = torch.as_tensor(synth.normal(c["seed"], 5000 + k, (R, bl, V)) * 3.0, dtype=torch.float32).cuda()
        sp = torch.empty(R, b, dtype=torch.int32, device="cuda")
        tk, sc = torch.empty_like(sp), torch.empty(R, b, dtype=torch.float32, device="cuda")
        st.beam_step(lg, sp, tk, sc)
        st.prune_compact(kp, vp)
        torch.cuda.synchronize()
        N = st.n_nodes.cpu().numpy()
        meta = [np.concatenate([x[r, : N[r]] for x in (st.token.cpu().numpy(), st.parent.cpu().numpy(),
                                                      st.depth.cpu().numpy(), st.beam_mask.cpu().numpy())])
                for r in range(R)]
        meta.append(st.leaf.cpu().numpy()[:, :b].ravel())
        metas = [None] * world
        dist.all_gather_object(metas, meta)
        same = all(len(m) == len(meta) and all(np.array_equal(a, b_) for a, b_ in zip(m, meta)) for m in metas)
        rec.append(dict(outs=outs, sp=sp.cpu().numpy(), tk=tk.cpu().numpy(), sc=sc.cpu().numpy(),
                        lg=lg.cpu().numpy(), same=same))
    status = st.status()
    if fg is not None:
        fg.close()
    dist.barrier()
    if rank == 0:
        q.put((rec, status))
    dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True], ids=["host-gather", "fused-peer-stores"])
def test_kv_head_shard_two_ranks_one_gpu_matches_oracle(fused):
    """fused=True: SURVEY §8(f) NEXT-4 -- the attention kernels store their output rows
    straight into both ranks' gather buffers (CUDA IPC on one GPU; peer-mapped over NVLink
    on a multi-GPU box) and trie_gather_wait hands back the all-head output."""
    need_gpu()
    import torch.multiprocessing as mp

    from oracle.kernels_ref import attn_ref, beam_step_ref
    from oracle.numerics import rope_rotate_half
    from oracle.trie import Trie, garbage_collect
    c = CFG
    R, b, t, Hq, Hkv, D, W, L, V, s = (c[k] for k in ("R", "b", "t", "Hq", "Hkv", "D", "W", "L", "V", "s"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, c, q, fused)) for r in range(2)]
    for p in procs:
        p.start()
    rec, status = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert status == 0
    prompts, lens = synth.prompts(c["seed"], R, t, V)
    tries = [Trie([int(x) for x in prompts[r][: lens[r]]], n_layers=L) for r in range(R)]
    for l in range(L):
        K0 = _bf(synth.normal(c["seed"], 10 + 2 * l, (R, Hkv, t, D))).float().numpy().astype(np.float64)
        V0 = _bf(synth.normal(c["seed"], 11 + 2 * l, (R, Hkv, t, D))).float().numpy().astype(np.float64)
        for r, T in enumerate(tries):
            T.kv[l] = [(K0[r][:, n], V0[r][:, n]) for n in range(T.t)]
    checked = 0
    for k, e in enumerate(rec):
        assert e["same"], f"step {k}: trie metadata differs between the ranks"
        bl = 1 if k == 0 else b
        for l in range(L):
            qf, kf, vf = (x.float().numpy().astype(np.float64) for x in _inputs(c, k, l, bl))
            for r, T in enumerate(tries):
                pos = T.depth[T.leaves[0]]
                for j, lf in enumerate(T.leaves):   # write before read (Alg. 3 l.7, §3.4)
                    T.kv[l][lf] = (rope_rotate_half(kf[r, j], pos, c["base"]), vf[r, j])
                Kr = np.stack([T.kv[l][n][0] for n in range(T.N)], axis=1)
                Vr = np.stack([T.kv[l][n][1] for n in range(T.N)], axis=1)
                qr = np.stack([rope_rotate_half(qf[r, j], pos, c["base"]) for j in range(bl)])
                o_ref, _ = attn_ref(qr, Kr, Vr, T, window=W)
                err = rel_err(e["outs"][l][r], o_ref)
                assert err <= 2e-2, f"step {k} layer {l} r={r}: gathered attention rel err {err:.3g}"
                checked += bl * Hq
        for r, T in enumerate(tries):
            refp, reft, refs, gap, _ = beam_step_ref(e["lg"][r][: len(T.leaves)], np.asarray(T.scores), b)
            if gap > 1e-5 * max(1.0, float(np.abs(refs).max())):
                assert e["sp"][r].tolist() == refp.tolist() and e["tk"][r].tolist() == reft.tolist()
            T.update_trie([(float(e["sc"][r, i]), int(e["tk"][r, i]), int(e["sp"][r, i])) for i in range(b)])
            garbage_collect(T)
    assert checked >= s * L * R * b * Hq // 2


@pytest.mark.parametrize("gather", ["fused", "host"])
def test_bench_kv_shard_two_ranks(gather):
    """bench.py --workload mistral-shard at N = 2 (two ranks on one GPU, eager gloo test
    mode): strong scaling, 4 of the 8 KV heads per rank, a per-layer all-gather -- fused
    into the attention kernels (NEXT-4, the default) or through host memory."""
    need_gpu()
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", BENCH_GATHER=gather)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
                          os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "mistral-shard",
                          "--requests", "2", "--steps", "4", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads([x for x in out.stdout.strip().splitlines() if x.startswith("{")][-1])
    assert res["n_gpus"] == 2 and res["value"] > 0 and res["scaling"] == "strong"
    assert res["config"]["kv_heads_per_gpu"] == 4 and res["config"]["q_heads_per_gpu"] == 16
    assert res["config"]["parallelism"].startswith("kv-head-shard2")
