"""Benchmark of the trie-decoding hot path on B200 (BASELINE.json metric).

One bench STEP = one beam-decode step of R requests through the whole hot path
(SURVEY §8(a) rows a-1..a-6): for every layer trie_rope_kv_append + trie_attn_decode,
then trie_beam_step (log-softmax + top-b + append + bitset update), then
trie_prune_compact (g = 1).  Jobs of s new tokens run back to back; when a job reaches s
steps the trie is re-initialised (trie_reset, inside the timed region) and the next job
starts from the resident prompts.  The model GEMMs are context, not product, and are
not in the step: Q/K/V and fp32 logits are seeded synthetic inputs resident in HBM
(`value`); `e2e` copies every step's Q/K/V + logits from pinned host memory and reads
back the selections (device-to-host) inside the timed region.

Metric (BASELINE.json): beam-decode steps/s (request-steps/s: one request advancing its
b beams by one token) and trie-attn HBM GB/s over unique-KV bytes (roofline object);
KV bytes vs batch beam search (kv_memory object).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload phi|llama|mistral-shard|sweep]
    python bench.py --impl reference ...   (the CPU oracle arm)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[1]: the N=1 metric workload
    "phi": dict(name="phi3.5-mini-mha-cnndm-t800-b4-s64", L=32, Hq=32, Hkv=32, D=96, V=32064,
                t=800, b=4, s=64, R=64, W=0, theta=10000.0),
    # configs[2]: request-parallel over 1/2/4/8 GPUs (R per GPU)
    "llama": dict(name="llama3.1-8b-gqa-humaneval-t150-b8-s256", L=32, Hq=32, Hkv=8, D=128,
                  V=128256, t=150, b=8, s=256, R=32, W=0, theta=500000.0),
    # configs[3], one rank's shard: 1 KV head + 4 query heads of 8, W = 4096 (reading A15)
    "mistral-shard": dict(name="mistral-small-24b-swa-t4096-b4-s128-kvshard1of8", L=40, Hq=4, Hkv=1,
                          D=128, V=131072, t=4096, b=4, s=128, R=16, W=4096, theta=1e8),
    # configs[4] kernel-level sweep point (b set by --beam)
    "sweep": dict(name="llama3.1-8b-gqa-t8192-sweep", L=4, Hq=32, Hkv=8, D=128, V=128256, t=8192,
                  b=16, s=128, R=4, W=0, theta=500000.0),
}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu_index: int):
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={gpu_index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7 and f[0].isdigit():
                rows.append(f)
        if not rows:
            return None
        sm = [int(r[0]) for r in rows]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][1]),
                "reasons": sorted(reasons), "samples": len(rows)}


# ------------------------------------------------------------------------------------------
def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2502_00085_b200 import _lib
    from paper_2502_00085_b200.build import build
    from paper_2502_00085_b200.trie import TrieState

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()
    _lib.load()
    dev = torch.device("cuda", local)
    wl = dict(WORKLOADS[args.workload])
    if args.beam:
        wl["b"] = args.beam
    if args.requests:
        wl["R"] = args.requests
    L, Hq, Hkv, D, V, t, b, s, R, W = (wl[k] for k in ("L", "Hq", "Hkv", "D", "V", "t", "b", "s", "R", "W"))
    cap = (t + b * s + b + 63) // 64 * 64  # whole 64-slot tiles (the TMA path needs cap % 4 == 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    import synth
    # request-parallel partition: rank owns requests [rank*R, (rank+1)*R) (weak scaling)
    prompts, lens = synth.prompts(10_000 + rank, R, t, V)
    st = TrieState(R, b, t, cap, L, Hq, Hkv, D, V, prompts, lens, window=W, dtype=torch.bfloat16,
                   device=dev)
    kp, vp = st.new_pools()
    for l in range(L):  # resident prompt K/V (prefill is model context; synthetic here)
        kp[l][:, :, :t].normal_(generator=gen)
        vp[l][:, :, :t].normal_(generator=gen)
    NB = 2
    qkv = [torch.randn(L, R, b, Hq + 2 * Hkv, D, device=dev, generator=gen).to(torch.bfloat16)
           for _ in range(NB)]
    NLOG = 8
    kappa = 3.0
    logits = [torch.randn(R, b, V, device=dev, generator=gen) * kappa for _ in range(NLOG)]
    q_l = [[x[l, :, :, :Hq].contiguous() for l in range(L)] for x in qkv]
    k_l = [[x[l, :, :, Hq:Hq + Hkv].contiguous() for l in range(L)] for x in qkv]
    v_l = [[x[l, :, :, Hq + Hkv:].contiguous() for l in range(L)] for x in qkv]
    # first step of every job has one live beam (the prompt leaf): separate contiguous inputs
    q1 = [[x[:, :1].contiguous() for x in ql] for ql in q_l]
    k1 = [[x[:, :1].contiguous() for x in kl] for kl in k_l]
    v1 = [[x[:, :1].contiguous() for x in vl] for vl in v_l]
    lg1 = [x[:, :1].contiguous() for x in logits]
    out = torch.empty(R, b, Hq, D, dtype=torch.bfloat16, device=dev)
    out1 = torch.empty(R, 1, Hq, D, dtype=torch.bfloat16, device=dev)
    sel_p = torch.empty(R, b, dtype=torch.int32, device=dev)
    sel_t = torch.empty_like(sel_p)
    sel_s = torch.empty(R, b, dtype=torch.float32, device=dev)
    rows_hint = t + s
    stream = torch.cuda.current_stream()
    attn_ev = []
    state = {"k": 0, "step": 0}

    def one_step(timed, qi, li, use_events):
        if state["k"] == s:
            st.reset()
            state["k"] = 0
        b_live = 1 if state["k"] == 0 else b
        for l in range(L):
            if b_live == 1:
                q, kk, vv, o = q1[qi][l], k1[qi][l], v1[qi][l], out1
            else:
                q, kk, vv, o = q_l[qi][l], k_l[qi][l], v_l[qi][l], out
            st.rope_kv_append(q, kk, vv, kp[l], vp[l], wl["theta"])
            if use_events:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            st.attn_decode(q, kp[l], vp[l], o, rows_hint=rows_hint)
            if use_events:
                e1.record(stream)
                attn_ev.append((e0, e1, b_live))
        lg = logits[li] if b_live == b else lg1[li]
        st.beam_step(lg, sel_p, sel_t, sel_s)
        st.prune_compact(kp, vp)
        state["k"] += 1
        state["step"] += 1

    # warm-up (untimed)
    for i in range(args.warmup):
        one_step(False, i % NB, i % NLOG, False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # N history for algorithmic-byte accounting
    n_hist = torch.empty(args.steps, R, dtype=torch.int32, device=dev)
    k_hist = []
    clocks = Clocks(local)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    launches0 = _lib.trie_launch_count()
    t0.record(stream)
    for i in range(args.steps):
        k_hist.append(state["k"] % s)
        n_hist[i].copy_(st.n_nodes, non_blocking=True)
        one_step(True, i % NB, i % NLOG, True)
    t1.record(stream)
    launches = _lib.trie_launch_count() - launches0
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    assert st.status() == 0, f"device status bits {st.status():#x}"
    # attention roofline
    attn_ms = [a.elapsed_time(bb) for a, bb, _ in attn_ev]
    nh = n_hist.cpu().numpy()
    bytes_attn = []
    for i in range(args.steps):
        after_reset = k_hist[i] == 0
        N = np.full(R, t) if after_reset else nh[i]
        bl = 1 if after_reset else b
        if W <= 0 or after_reset:
            U = N.astype(np.int64) if W <= 0 else np.full(R, min(t, W), np.int64)
        else:  # window lower depth = leaf depth - W + 1 = t + k - W (prompt part is a slot range)
            lo = max(0, t + k_hist[i] - W)
            U = (N - lo).astype(np.int64)
        kv = int(U.sum()) * 2 * Hkv * D * 2
        qo = R * bl * Hq * D * 2 * 2
        meta = int((N - t).clip(min=0).sum()) * 8
        bytes_attn += [kv + qo + meta] * L
    ach = float(np.sum(bytes_attn) / (np.sum(attn_ms) * 1e-3) / 1e9)
    peak, peak_src = _peaks()
    total_req_steps = R * args.steps * world
    value = total_req_steps / (ms * 1e-3)
    res = dict(metric="beam-decode steps/s (request-steps/s, hot path) + trie-attn HBM GB/s",
               value=round(value, 2), unit="request-steps/s", n_gpus=world, steps=args.steps,
               warmup=args.warmup, ms_per_step=round(ms / args.steps, 4), higher_is_better=True,
               scaling="weak", vs_baseline=None, dtype="bf16", data="synthetic",
               config=dict(workload=wl["name"], requests_per_gpu=R, beam=b, prompt_len=t,
                           new_tokens=s, layers=L, q_heads=Hq, kv_heads=Hkv, head_dim=D, vocab=V,
                           window=W, gc_interval=1, parallelism=f"request-dp{world}",
                           l2=(f"no flush: each layer's pool is re-read once per step and the "
                               f"per-step KV footprint ({R * t * Hkv * D * 4 * L / 1e6:.0f} MB) > L2 (126 MB)")))
    res["roofline"] = dict(kernel="trie_attn_decode", bound="hbm", achieved=round(ach, 1), peak=peak,
                           unit="GB/s", frac=round(ach / peak, 4), frac_of_8TBps=round(ach / 8000, 4),
                           traffic=None, peak_source=peak_src,
                           avg_launch_us=round(float(np.mean(attn_ms)) * 1e3, 2),
                           attn_share_of_step=round(float(np.sum(attn_ms)) / ms, 4))
    res["clocks"] = clk
    res["gpu_launches"] = int(launches)
    # KV memory vs batch beam search (logical bytes, SURVEY reading A18) at the timed step
    # that is deepest into its job: batch holds b * (t + k) rows per request (prompt
    # replicated, pending tokens included, P:42 counting); the trie holds N rows.
    i_star = int(np.argmax(k_hist))
    k_star = k_hist[i_star]
    kv_row = L * 2 * Hkv * D * 2
    trie_b = int(nh[i_star].sum()) * kv_row
    batch_b = R * (b if k_star > 0 else 1) * (t + k_star) * kv_row
    res["kv_memory"] = dict(step_in_job=int(k_star), trie_bytes=trie_b, batch_bytes=batch_b,
                            ratio_batch_over_trie=round(batch_b / max(trie_b, 1), 3),
                            bound_b_ts_over_t_s_b_1=round(b * (t + k_star) / (t + k_star + b - 1), 3))
    return res, dict(st=st, kp=kp, vp=vp, qkv=qkv, logits=logits, L=L, R=R, b=b, s=s, t=t, V=V,
                     world=world, rank=rank, dev=dev, wl=wl)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="phi", choices=sorted(WORKLOADS))
    ap.add_argument("--beam", type=int, default=0)
    ap.add_argument("--requests", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    res, ctx = run_gpu(args)
    if ctx["rank"] == 0:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
