"""Benchmark of the trie-decoding hot path on B200 (BASELINE.json metric).

One bench STEP = one beam-decode step of R requests through the whole hot path
(SURVEY §8(a) rows a-1..a-6): for every layer trie_rope_kv_append + trie_attn_decode,
then trie_beam_step (log-softmax + top-b + append + bitset update), then
trie_prune_compact (g = 1).  Jobs of s new tokens run back to back: the first step of a
job runs trie_reset + one live beam (the prompt leaf; its forward stands in for the
prefill's last position), the next s-1 steps run b live beams.  Steps are replayed as
CUDA graphs (one per input buffer x {first, steady}) so the host never paces the GPU.
The model GEMMs are context, not product, and are not in the step: Q/K/V and fp32 logits
are seeded synthetic inputs resident in HBM (`value`); `e2e` copies every step's Q/K/V +
logits from pinned host memory (double-buffered on a copy stream) and reads the step's
selections back to the host, all inside its timed region.

Metric (BASELINE.json): beam-decode steps/s (request-steps/s: one request advancing its
b beams by one token) and trie-attn HBM GB/s over unique-KV bytes (roofline object);
KV bytes vs batch beam search (kv_memory object).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload phi|llama|mistral-shard|sweep]
    python bench.py --impl reference ...   (the CPU oracle arm)
"""
from __future__ import annotations

import argparse
import json
import types
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[1]: the N=1 metric workload
    "phi": dict(name="phi3.5-mini-mha-cnndm-t800-b4-s64", L=32, Hq=32, Hkv=32, D=96, V=32064, d=3072, ffn=8192,
                t=800, b=4, s=64, R=64, W=0, theta=10000.0),
    # configs[2]: request-parallel over 1/2/4/8 GPUs (R per GPU)
    "llama": dict(name="llama3.1-8b-gqa-humaneval-t150-b8-s256", L=32, Hq=32, Hkv=8, D=128, d=4096, ffn=14336,
                  V=128256, t=150, b=8, s=256, R=32, W=0, theta=500000.0),
    # configs[3]: Mistral-Small-24B-shaped SWA, W = 4096 (reading A15); the 8 KV heads are
    # sharded over the N ranks (8/N KV heads + their 32/N query heads each, the SAME R
    # requests on every rank) with a per-layer all-gather of the attention outputs
    # (paper_2502_00085_b200/dist.py); strong scaling: the job is fixed, N = 1 holds all heads
    "mistral-shard": dict(name="mistral-small-24b-swa-t4096-b4-s128-kvshard", L=40, Hq=32, Hkv=8, d=5120, ffn=32768,
                          D=128, V=131072, t=4096, b=4, s=128, R=16, W=4096, theta=1e8, kv_shard=True),
    # configs[4] kernel-level sweep point (b set by --beam)
    "sweep": dict(name="llama3.1-8b-gqa-t8192-sweep", L=4, Hq=32, Hkv=8, D=128, V=128256, t=8192,
                  b=16, s=128, R=16, W=0, theta=500000.0),  # SURVEY cfg5: R in {1, 4, 16}
}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    QUERY = ("--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.gpu_index = gpu_index
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}_{gpu_index}.csv")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={gpu_index}", self.QUERY, "--format=csv,noheader,nounits",
                 "-lms", "100"],
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
        post = False
        if not rows:  # the sampler had not started writing yet: one query right at the end
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu_index}", self.QUERY,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=10).stdout
                rows = [[x.strip() for x in line.split(",")] for line in out.splitlines()
                        if line.strip() and line.split(",")[0].strip().isdigit()]
                post = True
            except Exception:
                rows = []
        if not rows:
            return None
        sm = [int(r[0]) for r in rows]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        res = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][1]),
               "reasons": sorted(reasons), "samples": len(rows)}
        if post:
            res["sampled"] = "once, right after the timed regions"
        return res


METRIC = "beam-decode steps/s (request-steps/s, hot path) + trie-attn HBM GB/s"


def _workload(args):
    wl = dict(WORKLOADS[args.workload])
    if args.beam:
        wl["b"] = args.beam
    if args.requests:
        wl["R"] = args.requests
    if getattr(args, "prompt_len", 0):
        wl["t"] = args.prompt_len
        wl["name"] += f"-t{args.prompt_len}"
    if getattr(args, "new_tokens", 0):
        wl["s"] = args.new_tokens
        wl["name"] += f"-s{args.new_tokens}"
    if getattr(args, "logit_scale", 0.0):
        wl["kappa"] = args.logit_scale
    if getattr(args, "paged", 0.0):
        wl["paged"] = args.paged
    wl["g"] = args.gc_interval
    wl["eos_frac"] = args.eos_frac
    return wl


def _scaling(wl):
    return "strong" if wl.get("kv_shard") else "weak"


def bench_config(wl, world):
    """The `config` object of the JSON line (both arms): the workload, per-GPU shape and
    parallelism (KV-head shard: each rank holds Hkv / world KV heads and their query heads)."""
    Hq, Hkv = wl["Hq"], wl["Hkv"]
    if wl.get("kv_shard"):
        Hq, Hkv = Hq // world, Hkv // world
    cfg = dict(workload=wl["name"], requests_per_gpu=wl["R"], beam=wl["b"], prompt_len=wl["t"],
               new_tokens=wl["s"], layers=wl["L"], q_heads_per_gpu=Hq, kv_heads_per_gpu=Hkv,
               head_dim=wl["D"], vocab=wl["V"], window=wl["W"], gc_interval=wl.get("g", 1),
               parallelism=(f"kv-head-shard{world} (per-layer all-gather of attention outputs)"
                            if wl.get("kv_shard") else f"request-dp{world}"))
    if wl.get("eos_frac"):
        cfg["eos_frac"] = wl["eos_frac"]
    if "kappa" in wl:
        cfg["logit_scale"] = wl["kappa"]
    if wl.get("paged"):
        cfg["kv_pool"] = f"paged (64-slot pages, prompt + {wl['paged']} x the no-GC generated pages)"
    return cfg


class _Eager:
    """Stand-in for a captured graph in the eager test mode: replay() re-runs the ops."""

    def __init__(self, fn):
        self.fn = fn

    def replay(self):
        self.fn()


# ------------------------------------------------------------------------------------------
class HotPath:
    """Buffers, trie state and captured step graphs for one rank."""

    def __init__(self, wl, rank, dev, world=1):
        import torch

        from paper_2502_00085_b200.trie import TrieState
        from paper_2502_00085_b200 import dist as tdist
        import synth
        self.torch = torch
        self.wl = wl
        L, Hq, Hkv, D, V, t, b, s, R, W = (wl[k] for k in ("L", "Hq", "Hkv", "D", "V", "t", "b", "s", "R", "W"))
        self.kv_shard = bool(wl.get("kv_shard"))
        self.world = world
        # eager test mode (BENCH_DIST_BACKEND=gloo, several ranks per GPU): the KV-head
        # shard's per-layer all-gather cannot be captured in a graph over gloo, so steps
        # run eagerly and the gather goes through host memory; the driver's runs are NCCL
        self.eager = self.kv_shard and world > 1 and os.environ.get("BENCH_DIST_BACKEND", "nccl") != "nccl"
        if self.kv_shard:  # this rank's KV heads and their query heads
            _, Hkv, _, Hq = tdist.kv_head_shard(Hq, Hkv, world, rank)
        self.L, self.Hq, self.Hkv, self.D, self.V, self.t, self.b, self.s, self.R, self.W = \
            L, Hq, Hkv, D, V, t, b, s, R, W
        self.cap = (t + b * s + b + 63) // 64 * 64  # whole 64-slot tiles (TMA path: cap % 4 == 0)
        self.dev = dev
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234 + rank)
        # logits drive the beam step: identical on every rank of a KV-head shard (same
        # requests, same selections, same trie metadata)
        lgen = torch.Generator(device=dev)
        lgen.manual_seed(4321 + (0 if self.kv_shard else rank))
        # request-parallel partition: this rank owns its own R requests (weak scaling);
        # KV-head shard: every rank holds the same R requests
        prompts, lens = synth.prompts(10_000 + (0 if self.kv_shard else rank), R, t, V)
        # NEXT-2 (--paged f): paged pools of 64-slot pages -- the prompt's pages plus f x the
        # no-GC worst case of generated pages, shared by all requests (pages are mapped as a
        # trie grows and returned by GC; TRIE_ST_CAPACITY latches if the pool runs dry)
        self.n_pages = 0
        if wl.get("paged"):
            self.n_pages = R * ((t + 63) // 64 + int(np.ceil(wl["paged"] * (b * s + b) / 64)) + 1)
        self.st = TrieState(R, b, t, self.cap, L, Hq, Hkv, D, V, prompts, lens, window=W,
                            dtype=torch.bfloat16, device=dev, n_pages=self.n_pages)
        self.kp, self.vp = self.st.new_pools()
        for l in range(L):  # resident prompt K/V (prefill is model context; synthetic here)
            if self.n_pages:  # the prompt pages are the first R * ceil(t / 64) pages
                self.kp[l][: R * ((t + 63) // 64)].normal_(generator=gen)
                self.vp[l][: R * ((t + 63) // 64)].normal_(generator=gen)
            else:
                self.kp[l][:, :, :t].normal_(generator=gen)
                self.vp[l][:, :, :t].normal_(generator=gen)
        # inputs: 2 slots x {first (1 live beam), steady (b live beams)}; one flat buffer each
        self.NB = 2
        self.inp = {}
        for var, bl in (("first", 1), ("steady", b)):
            per_layer = R * bl * (Hq + 2 * Hkv) * D
            for slot in range(self.NB):
                qkv = torch.randn(L * per_layer, device=dev, generator=gen).to(torch.bfloat16)
                lg = torch.randn(R * bl * V, device=dev, generator=lgen) * float(wl.get("kappa", 3.0))
                if wl.get("eos_frac", 0.0) > 0.0 and var == "steady":
                    # NEXT-3 experiment (--eos-frac f): EOS (token 0) is the argmax of every
                    # row of the first round(f R) requests, so they finish at their second
                    # step and are done from the third on; the others never emit it
                    nf = int(round(wl["eos_frac"] * R))
                    lg3 = lg.view(R, bl, V)
                    lg3[:nf, :, 0] = lg3[:nf].amax(dim=-1) + 30.0
                    lg3[nf:, :, 0] = -30.0
                views = []
                for l in range(L):
                    base = l * per_layer
                    q = qkv[base: base + R * bl * Hq * D].view(R, bl, Hq, D)
                    k = qkv[base + R * bl * Hq * D: base + R * bl * (Hq + Hkv) * D].view(R, bl, Hkv, D)
                    v = qkv[base + R * bl * (Hq + Hkv) * D: base + per_layer].view(R, bl, Hkv, D)
                    views.append((q, k, v))
                self.inp[(var, slot)] = dict(qkv=qkv, logits=lg.view(R, bl, V), views=views,
                                             out=torch.empty(R, bl, Hq, D, dtype=torch.bfloat16, device=dev))
        # all-gather target of the attention outputs (KV-head shard, N > 1)
        self.gathered = (torch.empty(world, R, b, Hq, D, dtype=torch.bfloat16, device=dev)
                         if self.kv_shard and world > 1 else None)
        self.gathered1 = (torch.empty(world, R, 1, Hq, D, dtype=torch.bfloat16, device=dev)
                          if self.gathered is not None else None)
        # NEXT-4 (default for the KV-head shard at N > 1): the all-gather fused into the
        # attention kernels -- peer stores from the epilogue into every rank's gather buffer
        # (CUDA IPC / NVLink), a flag per rank, trie_gather_wait; BENCH_GATHER=nccl keeps the
        # NCCL all_gather_into_tensor per layer instead
        self.fg = None
        if self.gathered is not None and os.environ.get("BENCH_GATHER", "fused") == "fused":
            self.fg = tdist.FusedGather(self.st, world, rank)
            self.gathered = torch.empty(R, b, world * Hq, D, dtype=torch.bfloat16, device=dev)
            self.gathered1 = torch.empty(R, 1, world * Hq, D, dtype=torch.bfloat16, device=dev)
        self.sel_p = torch.empty(R, b, dtype=torch.int32, device=dev)
        self.sel_t = torch.empty_like(self.sel_p)
        self.sel_s = torch.empty(R, b, dtype=torch.float32, device=dev)
        self.rows_hint = t + s
        if wl.get("eos_frac", 0.0) > 0.0:
            self.st.set_eos(0)
        self.g = int(wl.get("g", 1))  # GC interval (Alg. 2); 1 on the hot path
        self.graphs = {}
        self.launches_per_graph = {}
        self.k = 0  # steps done in the current job
        from paper_2502_00085_b200 import _lib
        self.plan = {var: _lib.trie_attn_plan_info(self.st.cfg, bl, self.rows_hint)
                     for var, bl in (("first", 1), ("steady", b))}
        # a-1 + a-3 as one trie_attn_decode_rope launch per layer wherever the plan has a
        # fused kernel (narrow / wide): measured r27, request-steps/s fused vs two launches:
        # Llama 52,301 vs 48,464, Phi 17,309 vs 17,062.  TRIE_BENCH_FUSED=0 forces two launches.
        self.fused = {var: self.plan[var]["fused_rope"] and os.environ.get("TRIE_BENCH_FUSED") != "0"
                      for var in self.plan}

    def step_ops(self, var, slot, events=None, gc=True):
        """Enqueue one step (all §8(a) rows) on the current stream; `gc` = run a-6 after
        the append (Alg. 2 l.5-7 with interval g: the bench's gc_now())."""
        st, L = self.st, self.L
        d = self.inp[(var, slot)]
        if var == "first":
            st.reset()
        fused = self.fused[var]
        if events is not None and fused:  # the layer loop is L attention launches only
            events[0][0].record()
        for l in range(L):
            q, k, v = d["views"][l]
            if fused:  # a-1 + a-3 in one launch
                st.attn_decode_rope(q, k, v, self.kp[l], self.vp[l], self.wl["theta"], d["out"],
                                    rows_hint=self.rows_hint)
                if self.gathered is not None:
                    self._gather(d["out"])
                continue
            st.rope_kv_append(q, k, v, self.kp[l], self.vp[l], self.wl["theta"])
            if events is not None:
                events[l][0].record()
            st.attn_decode(q, self.kp[l], self.vp[l], d["out"], rows_hint=self.rows_hint)
            if events is not None:
                events[l][1].record()
            if self.gathered is not None:  # KV-head shard: every rank needs every head
                self._gather(d["out"])
        if events is not None and fused:
            events[0][1].record()
        if events is not None:  # the last two pairs: beam step (a-4/a-5/a-2), GC (a-6)
            events[-2][0].record()
        st.beam_step(d["logits"], self.sel_p, self.sel_t, self.sel_s)
        if events is not None:
            events[-2][1].record()
            events[-1][0].record()
        if gc:
            st.prune_compact(self.kp, self.vp)
        if events is not None:
            events[-1][1].record()

    def _gather(self, out):
        from paper_2502_00085_b200.dist import gather_heads
        # the first step of a job has one live beam: its own buffer
        dst = self.gathered if out.shape[1] == self.b else self.gathered1
        if self.fg is not None:  # fused: the kernel already stored into every rank's buffer
            self.fg.wait(dst)
            return
        if self.eager:  # gloo: through host memory
            dst.copy_(gather_heads(out.cpu()))
            return
        gather_heads(out, dst)

    def capture(self):
        """One graph per (variant, slot) + an event-instrumented twin for kernel timing."""
        torch = self.torch
        from paper_2502_00085_b200 import _lib
        self.ev = {}
        gcs = (True,) if self.g == 1 else (True, False)
        for var in ("first", "steady"):
            for slot in range(self.NB):
                for gc in gcs:
                    for timed in (False, True):
                        evs = None
                        if timed:
                            n_pairs = (1 if self.fused[var] else self.L) + 2
                            evs = [(torch.cuda.Event(enable_timing=True, external=True),
                                    torch.cuda.Event(enable_timing=True, external=True))
                                   for _ in range(n_pairs)]
                        key = ((var, gc), slot, timed)
                        if self.eager:
                            self.graphs[key] = _Eager(
                                lambda var=var, slot=slot, evs=evs, gc=gc: self.step_ops(var, slot, evs, gc))
                            self.launches_per_graph[key] = None  # counted at run time
                            if timed:
                                self.ev[((var, gc), slot)] = evs
                            continue
                        g = torch.cuda.CUDAGraph()
                        n0 = _lib.trie_launch_count()
                        with torch.cuda.graph(g):
                            self.step_ops(var, slot, evs, gc)
                        self.graphs[key] = g
                        self.launches_per_graph[key] = _lib.trie_launch_count() - n0
                        if timed:
                            self.ev[((var, gc), slot)] = evs
        # capture ran the host logic of reset/beam_step: the host view is at "steady" (b
        # live beams) now, so the roofline's attention-only graph is captured here
        self._capture_attn_only()

    def _capture_attn_only(self):
        """Region C's graph: the step's L attention launches (fused a-1 + a-3 where planned)
        on the steady inputs, with b live beams -- the handle's host view right after the
        steady step graphs were captured (a later trie_reset sets it back to one beam)."""
        torch = self.torch
        st, L = self.st, self.L
        d = self.inp[("steady", 0)]
        if self.eager:  # the host view is still at its warm-up state: b live beams after step 1
            def attn_only():
                for l in range(L):
                    q, k, v = d["views"][l]
                    if self.fused["steady"]:
                        st.attn_decode_rope(q, k, v, self.kp[l], self.vp[l], self.wl["theta"], d["out"],
                                            rows_hint=self.rows_hint)
                    else:
                        st.attn_decode(q, self.kp[l], self.vp[l], d["out"], rows_hint=self.rows_hint)
            self.attn_graph = _Eager(attn_only)
            return
        assert st.b_live == self.b, "attention-only graph must be captured with b live beams"
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for l in range(L):
                q, k, v = d["views"][l]
                if self.fused["steady"]:  # idempotent: q is read, the leaves' rows re-written
                    st.attn_decode_rope(q, k, v, self.kp[l], self.vp[l], self.wl["theta"], d["out"],
                                        rows_hint=self.rows_hint)
                else:
                    st.attn_decode(q, self.kp[l], self.vp[l], d["out"], rows_hint=self.rows_hint)
        self.attn_graph = g

    def gc_now(self, k=None):
        """GC after the append of job step k (0-based) iff Alg. 2's top-of-iteration test
        i mod g == 0 holds at i = t + k + 1 (readings R7 / R8); g = 0: never."""
        k = self.k if k is None else k
        return self.g == 1 or (self.g > 1 and (self.t + k + 1) % self.g == 0)

    def next_key(self):
        var = "first" if self.k % self.s == 0 else "steady"
        return (var, self.gc_now())

    def replay(self, slot, timed=False):
        key = self.next_key()
        self.graphs[(key, slot, timed)].replay()
        self.k = (self.k + 1) % self.s
        return key

    def attn_only_timing(self, reps=10):
        """Mean duration (us) and algorithmic bytes of one trie_attn_decode launch: the
        graph of the L layers' steady launches (captured with the step graphs), replayed
        `reps` times on the trie the timed steps left."""
        torch = self.torch
        L = self.L
        if self.k == 0:  # a job boundary: the trie holds only the prompt; step once
            self.replay(0)
        torch.cuda.synchronize()
        g = self.attn_graph
        g.replay()
        if os.environ.get("BENCH_PROFILE_REGION_C"):
            # ncu --profile-from-start off: exactly one replay of region C's launches (the
            # roofline's trie state) is profiled (scripts/ncu_region_c.sh)
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
            g.replay()
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
        done = None
        if self.wl.get("eos_frac"):  # NEXT-3: requests whose beams all finished are skipped
            done = (self.st.finished.cpu().numpy()[:, :self.b] != 0).all(axis=1)
        torch.cuda.synchronize()
        # one event per replay boundary (back to back, no host sync in between): the mean
        # over all reps * L launches, and the spread of the per-replay means
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        evs[0].record()
        for i in range(reps):
            g.replay()
            evs[i + 1].record()
        torch.cuda.synchronize()
        per = np.array([evs[i].elapsed_time(evs[i + 1]) * 1e3 / L for i in range(reps)])
        us = evs[0].elapsed_time(evs[-1]) * 1e3 / (reps * L)
        self.attn_spread = dict(replays=reps, launches=reps * L,
                                p10_us=round(float(np.percentile(per, 10)), 2),
                                median_us=round(float(np.median(per)), 2),
                                p90_us=round(float(np.percentile(per, 90)), 2))
        return us, self.attn_bytes(self.k, self.live_rows(), None if done is None else ~done)

    def live_rows(self):
        """Per request: rows some live beam can see (prompt + generated nodes with a
        beam bit).  With GC every step this is N; with g > 1 dead rows (mask 0) are not
        algorithmic bytes although the kernel still streams them."""
        N = self.st.n_nodes.cpu().numpy()
        if self.g == 1:
            return N
        m = self.st.beam_mask.cpu().numpy()
        t = self.st.prompt_len.cpu().numpy()
        return np.array([t[r] + int(np.count_nonzero(m[r, t[r]:N[r]])) for r in range(self.R)])

    def attn_bytes(self, k_in_job, N, live=None):
        """Algorithmic bytes of one trie_attn_decode launch: unique
        KV rows U_r x 2*Hkv*D*2 + Q and O (bf16) + mask/depth words of generated rows.
        live: optional [R] bool -- requests still decoding (NEXT-3: done requests, all
        beams finished at EOS, are skipped by the kernels and move no bytes)."""
        t, b, W, R, Hq, Hkv, D = self.t, self.b, self.W, self.R, self.Hq, self.Hkv, self.D
        if live is not None and not np.all(live):
            sub = types.SimpleNamespace(t=t, b=b, W=W, R=int(np.sum(live)), Hq=Hq, Hkv=Hkv, D=D)
            return HotPath.attn_bytes(sub, k_in_job, np.asarray(N)[np.asarray(live, bool)])
        bl = 1 if k_in_job == 0 else b
        if k_in_job == 0:
            N = np.full(R, t)
        if W <= 0:
            U = N.astype(np.int64)
        else:  # window lower depth = leaf depth - W + 1 (leaves share depth t + k - 1)
            leaf_depth = t - 1 if k_in_job == 0 else t + k_in_job - 1
            lo = max(0, leaf_depth - W + 1)
            U = (N - min(lo, t)).astype(np.int64)
        return int(U.sum()) * 2 * Hkv * D * 2 + R * bl * Hq * D * 2 * 2 + int((N - t).clip(min=0).sum()) * 8


class BatchPath:
    """SURVEY §8(f) NEXT-2 baseline: conventional batch beam search (Alg. 1) on
    the GPU with the same kernels, for the trie-vs-batch comparison on B200.  Every beam
    owns a private cache holding the whole prompt (replicated b times): a
    handle of R*b single-beam chains whose fused RoPE + append + attention launch reads each
    beam's own t+k rows; the top-b is the same trie_beam_step kernel (on a selection-only
    handle); after it, every beam's cache becomes a copy of its parent beam's (Alg. 1
    l.6-7; HF _reorder_cache): trie_batch_reorder_kv between two pool sets (ping-pong),
    copying the generated rows (the identical prompt rows are not copied -- this favours
    the baseline).  No GC: batch search never frees rows."""

    def __init__(self, wl, dev):
        import torch

        from paper_2502_00085_b200.trie import TrieState
        import synth
        self.torch = torch
        self.wl = wl
        L, Hq, Hkv, D, V, t, b, s, R = (wl[k] for k in ("L", "Hq", "Hkv", "D", "V", "t", "b", "s", "R"))
        self.L, self.Hq, self.Hkv, self.D, self.V, self.t, self.b, self.s, self.R = L, Hq, Hkv, D, V, t, b, s, R
        self.cap = (t + s + 1 + 63) // 64 * 64
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234)
        lgen = torch.Generator(device=dev)
        lgen.manual_seed(4321)
        prompts, lens = synth.prompts(10_000, R, t, V)
        self.chains = TrieState(R * b, 1, t, self.cap, L, Hq, Hkv, D, V, np.repeat(prompts, b, axis=0),
                                np.repeat(lens, b), dtype=torch.bfloat16, device=dev)
        self.sel = TrieState(R, b, t, (t + b * s + b + 63) // 64 * 64, 0, Hq, Hkv, D, V, prompts, lens,
                             dtype=torch.bfloat16, device=dev)
        # two pool sets (the reorder is out of place); prompt rows replicated per beam
        self.P = [self.chains.new_pools() for _ in range(2)]
        for l in range(L):
            pk = torch.randn(R, 1, Hkv, t, D, device=dev, generator=gen).to(torch.bfloat16)
            pv = torch.randn(R, 1, Hkv, t, D, device=dev, generator=gen).to(torch.bfloat16)
            for kp, vp in self.P:
                kp[l].view(R, b, Hkv, self.cap, D)[:, :, :, :t] = pk
                vp[l].view(R, b, Hkv, self.cap, D)[:, :, :, :t] = pv
        per_layer = R * b * (Hq + 2 * Hkv) * D
        self.qkv = torch.randn(L * per_layer, device=dev, generator=gen).to(torch.bfloat16)
        self.views = []
        for l in range(L):
            base = l * per_layer
            q = self.qkv[base: base + R * b * Hq * D].view(R * b, 1, Hq, D)
            k = self.qkv[base + R * b * Hq * D: base + R * b * (Hq + Hkv) * D].view(R * b, 1, Hkv, D)
            v = self.qkv[base + R * b * (Hq + Hkv) * D: base + per_layer].view(R * b, 1, Hkv, D)
            self.views.append((q, k, v))
        self.out = torch.empty(R * b, 1, Hq, D, dtype=torch.bfloat16, device=dev)
        self.logits = {"first": torch.randn(R, 1, V, device=dev, generator=lgen) * 3.0,
                       "steady": torch.randn(R, b, V, device=dev, generator=lgen) * 3.0}
        self.sel_p = torch.empty(R, b, dtype=torch.int32, device=dev)
        self.sel_t = torch.empty_like(self.sel_p)
        self.sel_s = torch.empty(R, b, dtype=torch.float32, device=dev)
        self.zeros = torch.zeros(R * b, dtype=torch.int32, device=dev)
        self.graphs = {}
        self.launches = {}
        self.k = 0

    def pool_bytes(self):
        return 2 * 2 * self.L * self.R * self.b * self.Hkv * self.cap * self.D * 2

    def step_ops(self, var, cur):
        from paper_2502_00085_b200 import _lib
        ch, se = self.chains, self.sel
        if var == "first":
            ch.reset()
            se.reset()
        kp, vp = self.P[cur]
        for l in range(self.L):
            q, k, v = self.views[l]
            ch.attn_decode_rope(q, k, v, kp[l], vp[l], self.wl["theta"], self.out, rows_hint=self.t + self.s)
        se.beam_step(self.logits[var], self.sel_p, self.sel_t, self.sel_s)
        nk, nv = self.P[1 - cur]
        _lib.trie_batch_reorder_kv(self.R, self.b, self.Hkv, self.D, self.cap, self.sel_p, ch.prompt_len,
                                   ch.n_nodes, [kp[l] for l in range(self.L)], [vp[l] for l in range(self.L)],
                                   [nk[l] for l in range(self.L)], [nv[l] for l in range(self.L)])
        ch.append(self.zeros, self.sel_t.view(-1))

    def capture(self):
        from paper_2502_00085_b200 import _lib
        torch = self.torch
        for var, cur in (("first", 0), ("steady", 1), ("steady", 0)):
            g = torch.cuda.CUDAGraph()
            n0 = _lib.trie_launch_count()
            with torch.cuda.graph(g):
                self.step_ops(var, cur)
            self.graphs[(var, cur)] = g
            self.launches[(var, cur)] = _lib.trie_launch_count() - n0

    def replay(self):
        key = ("first" if self.k == 0 else "steady", self.k % 2)
        self.graphs[key].replay()
        self.k = (self.k + 1) % self.s
        return key


def run_batch(args):
    """--impl batch: the NEXT-2 GPU batch-beam-search baseline on the same workload (one GPU;
    R halved until the two per-beam pool sets fit in 70% of free memory)."""
    import torch

    from paper_2502_00085_b200 import _lib
    from paper_2502_00085_b200.build import build
    build()
    _lib.load()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    wl = dict(WORKLOADS[args.workload])
    if args.beam:
        wl["b"] = args.beam
    if args.requests:
        wl["R"] = args.requests
    if wl.get("W", 0) or wl.get("kv_shard"):
        raise SystemExit("--impl batch: dense, unsharded workloads only")
    free = torch.cuda.mem_get_info()[0]
    while wl["R"] > 1:
        cap = (wl["t"] + wl["s"] + 1 + 63) // 64 * 64
        need = 2 * 2 * wl["L"] * wl["R"] * wl["b"] * wl["Hkv"] * cap * wl["D"] * 2
        if need <= 0.7 * free:
            break
        wl["R"] //= 2
    bp = BatchPath(wl, dev)
    for i in range(2):
        bp.step_ops("first" if i == 0 else "steady", i % 2)
    torch.cuda.synchronize()
    bp.capture()
    bp.k = 0
    for _ in range(args.warmup):
        bp.replay()
    if args.steps < bp.s:  # the same mid-job window as the trie arm (run_gpu)
        while bp.k != (bp.s - args.steps) // 2:
            bp.replay()
    torch.cuda.synchronize()
    clocks = Clocks(0)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k_hist, launches = [], 0
    t0.record()
    for _ in range(args.steps):
        k_hist.append(bp.k)
        launches += bp.launches[bp.replay()]
    t1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    st = bp.chains.status() | bp.sel.status()
    assert st == 0, f"device status bits {st:#x}"
    R, b, t, L = bp.R, bp.b, bp.t, bp.L
    kv_row = L * 2 * bp.Hkv * bp.D * 2
    k_mean = float(np.mean(k_hist))
    res = dict(metric="beam-decode steps/s (request-steps/s): GPU batch beam search baseline (NEXT-2)",
               value=round(R * args.steps / (ms * 1e-3), 2), unit="request-steps/s", n_gpus=1,
               steps=args.steps, warmup=args.warmup, ms_per_step=round(ms / args.steps, 4),
               higher_is_better=True, scaling="weak", vs_baseline=None, dtype="bf16", data="synthetic",
               impl="batch",
               config=dict(workload=wl["name"], requests_per_gpu=R, beam=b, prompt_len=t, new_tokens=bp.s,
                           layers=L, q_heads_per_gpu=bp.Hq, kv_heads_per_gpu=bp.Hkv, head_dim=bp.D,
                           vocab=bp.V, execution="cuda-graph replay per step",
                           algorithm="Alg. 1: b private caches per request (prompt replicated), per-beam "
                                     "attention over t+k rows, same top-b kernel, cache reorder by copy "
                                     "(generated rows; prompt rows not copied) into a second pool set"),
               kv_memory=dict(logical_bytes_mean=int(R * b * (t + k_mean) * kv_row),
                              physical_pool_bytes=int(bp.pool_bytes())),
               execution=dict(timed_job_steps=[int(k_hist[0]), int(k_hist[-1])]),
               clocks=clk, gpu_launches=int(launches))
    return res


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2502_00085_b200 import _lib
    from paper_2502_00085_b200.build import build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_DIST_BACKEND=gloo + several ranks per GPU is a test mode for boxes with fewer
    # GPUs than ranks (the driver's runs use NCCL, one rank per GPU)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if world > 1:
        dist.init_process_group(backend)
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()
    _lib.load()
    dev = torch.device("cuda", local)
    wl = _workload(args)
    hp = HotPath(wl, rank, dev, world)
    R, L, s, b, t = hp.R, hp.L, hp.s, hp.b, hp.t

    # eager warm-up (allocates scratch, sets kernel attributes), then capture
    for i in range(2):
        hp.step_ops("first" if i == 0 else "steady", i % 2, gc=hp.gc_now(i))
    torch.cuda.synchronize()
    hp.capture()
    hp.st.reset()
    torch.cuda.synchronize()
    hp.k = 0
    for i in range(args.warmup):
        hp.replay(i % 2)
    # untimed positioning replays: the K timed steps cover the MIDDLE of a job (job steps
    # k0 .. k0+K-1 with k0 = (s - K) / 2) so a short run is not biased to the small tries
    # of a job's start; K >= s covers whole jobs from wherever the warm-up left off
    n_pos = 0
    if args.steps < s:
        k0 = (s - args.steps) // 2
        while hp.k != k0:
            hp.replay((args.warmup + n_pos) % 2)
            n_pos += 1
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    stream = torch.cuda.current_stream()
    n_hist = torch.empty(args.steps, R, dtype=torch.int32, device=dev)
    k_hist = []
    launches = 0
    clocks = Clocks(local)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    # Timed region: instrumented step graphs (event nodes around every attention launch).
    # Slot i%2's events are harvested just before that slot's graph is replayed again
    # (step i+2): the host waits only for step i's end event, so step i+1 keeps the GPU busy.
    attn_ms, attn_bytes = [], []
    pending = {}
    end_ev = [torch.cuda.Event() for _ in range(2)]

    attn_step = []  # (step index, k in job) per harvested launch; bytes computed afterwards
    beam_ms, gc_ms = [], []  # per instrumented step: trie_beam_step, trie_prune_compact

    def harvest(slot):
        var_p, kj_p, i_p = pending.pop(slot)
        end_ev[slot].synchronize()  # only step i_p; step i_p + 1 keeps the GPU busy
        evs = hp.ev[(var_p, slot)]  # var_p = (variant, gc) key
        per = hp.L // (len(evs) - 2)  # fused: one pair spans the L attention launches of the step
        for e0, e1 in evs[:-2]:
            dt = e0.elapsed_time(e1)
            for _ in range(per):
                attn_ms.append(dt / per)
                attn_step.append((i_p, kj_p))
        beam_ms.append(evs[-2][0].elapsed_time(evs[-2][1]))
        gc_ms.append(evs[-1][0].elapsed_time(evs[-1][1]))

    # Region A (value): plain step graphs back to back.
    t0.record(stream)
    n_launch0 = _lib.trie_launch_count()  # eager mode: host-side launch counter
    for i in range(args.steps):
        k_hist.append(hp.k)
        n_hist[i].copy_(hp.st.n_nodes, non_blocking=True)  # 4*R bytes, for byte accounting
        var = hp.replay(i % 2)
        if not hp.eager:
            launches += hp.launches_per_graph[(var, i % 2, False)]
    if hp.eager:
        launches = _lib.trie_launch_count() - n_launch0
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    def advance_to(kt):  # untimed plain replays up to job step kt (the next job's if passed)
        while hp.k != kt:
            hp.replay(0)
    kA = k_hist[0] if args.steps < s else None
    # Region C (roofline): the L attention launches of one step (steady beams) as one graph
    # of back-to-back launches, replayed between CUDA events on the launching stream --
    # kernel time without the event-node latency that region B's per-launch events add --
    # on the trie at the MIDDLE of region A's window (same job step, next job)
    if kA is not None:
        advance_to((kA + args.steps // 2) % s)
    c_us, c_bytes = hp.attn_only_timing(reps=max(4, min(20, 2 * args.steps)))
    k_c = hp.k
    # Region B (roofline): region A's window again (same job steps, next job) with the
    # instrumented graphs (event nodes around every attention launch; event-record nodes
    # add ~5 us of graph latency each, so they are kept out of region A).  Slot i%2's
    # events are harvested just before that slot is replayed again, waiting only for that
    # step's end event.
    if kA is not None:
        advance_to(kA)
    n_hist_b = torch.empty(args.steps, R, dtype=torch.int32, device=dev)
    t2 = torch.cuda.Event(enable_timing=True)
    t3 = torch.cuda.Event(enable_timing=True)
    t2.record(stream)
    for i in range(args.steps):
        slot = i % 2
        if slot in pending:
            harvest(slot)
        n_hist_b[i].copy_(hp.st.n_nodes, non_blocking=True)
        kj = hp.k
        var = hp.replay(slot, timed=True)
        end_ev[slot].record(stream)
        pending[slot] = (var, kj, i)
    t3.record(stream)
    torch.cuda.synchronize()
    for slot in list(pending):
        harvest(slot)
    ms_b = t2.elapsed_time(t3)
    nh_all = n_hist_b.cpu().numpy()
    def live_at(kj):  # NEXT-3 experiment: the first round(f R) requests are done from job step 2
        if not wl.get("eos_frac") or kj < 2:
            return None
        lv = np.ones(R, bool)
        lv[: int(round(wl["eos_frac"] * R))] = False
        return lv
    attn_bytes = [hp.attn_bytes(kj, nh_all[i], live_at(kj)) for i, kj in attn_step]
    st_bits = hp.st.status()
    assert st_bits == 0, f"device status bits {st_bits:#x}"
    in_step_gbs = float(np.sum(attn_bytes) / (np.sum(attn_ms) * 1e-3) / 1e9)
    # clocks sampled across regions A, B and C (contiguous GPU work, 100 ms period)
    clk = clocks.stop()
    ach = c_bytes / (c_us * 1e-6) / 1e9
    peak, peak_src = _peaks()

    # request-DP: every rank its own R requests; KV-head shard: the same R on every rank
    units = R if hp.kv_shard else R * world
    value = units * args.steps / (ms * 1e-3)
    kv_fp = R * (t + s // 2) * hp.Hkv * hp.D * 4 * L
    res = dict(metric=METRIC, value=round(value, 2), unit="request-steps/s", n_gpus=world, steps=args.steps,
               warmup=args.warmup, ms_per_step=round(ms / args.steps, 4), higher_is_better=True,
               scaling=_scaling(wl), vs_baseline=None, dtype="bf16", data="synthetic",
               config=bench_config(wl, world),
               execution=dict(steps=("eager (gloo test mode: host-memory all-gather)" if hp.eager
                                     else "cuda-graph replay per step"),
                              attention={k: v for k, v in hp.plan["steady"].items()},
                              l2=(f"no flush: each layer's pool is re-read once per step and the per-step "
                                  f"KV footprint ({kv_fp / 1e6:.0f} MB) > L2 (126 MB)")))
    res["roofline"] = dict(kernel="trie_attn_decode", bound="hbm", achieved=round(ach, 1), peak=peak,
                           unit="GB/s", frac=round(ach / peak, 4), frac_of_8TBps=round(ach / 8000, 4),
                           traffic=_traffic(args.workload, R, b), peak_source=peak_src,
                           avg_launch_us=round(c_us, 2), bytes_per_launch=int(c_bytes),
                           launch_us_spread=hp.attn_spread,
                           kernel_launch=("trie_attn_decode_rope (fused a-1 + a-3; bytes counted: a-3 only)"
                                          if hp.fused["steady"] else "trie_attn_decode"),
                           timing=(f"CUDA events around a graph of the step's {hp.L} attention launches "
                                   f"(one per layer, back to back, at step {k_c} of a job: the middle of "
                                   f"the timed window), replayed after the timed steps; achieved = "
                                   f"algorithmic bytes / mean launch time"),
                           in_step=dict(achieved=round(in_step_gbs, 1),
                                        avg_launch_us=round(float(np.mean(attn_ms)) * 1e3, 2),
                                        attn_share_of_step=round(float(np.sum(attn_ms)) / ms_b, 4),
                                        breakdown_ms_per_step=dict(
                                            attn=round(float(np.sum(attn_ms)) / args.steps, 4),
                                            beam_step=round(float(np.mean(beam_ms)), 4),
                                            gc=round(float(np.mean(gc_ms)), 4),
                                            step=round(ms_b / args.steps, 4),
                                            note="region B event nodes (they also break the PDL chain, "
                                                 "so the short beam-step / gc intervals read high: "
                                                 "scripts/gc_cost.py measures gc without them); the "
                                                 "model GEMMs are context and not in the step (SURVEY §8(d))"),
                                        timing="CUDA event nodes around every attention launch of "
                                               f"{args.steps} instrumented step graphs "
                                               f"({ms_b / args.steps:.3f} ms/step; includes the "
                                               "event nodes' launch latency)"))
    if hp.n_pages:  # NEXT-2: the physical peak (the paper's allocator-peak metric)
        ps = hp.st.page_stats()
        page_bytes = 64 * L * 2 * hp.Hkv * hp.D * 2
        res["paged_pool"] = dict(n_pages=ps["n_pages"], peak_pages=ps["peak"], in_use_end=ps["in_use"],
                                 page_bytes_all_layers=page_bytes, peak_bytes=ps["peak"] * page_bytes,
                                 batch_physical_bytes=R * b * hp.cap * L * 2 * hp.Hkv * hp.D * 2,
                                 note="peak pages in use since trie_create (device counter), i.e. over every job of the run; "
                                      "batch = b private caches of t + s rows per request")
    res["clocks"] = clk
    res["gpu_launches"] = int(launches)
    nh = n_hist.cpu().numpy()
    i_star = int(np.argmax(k_hist))
    k_star = k_hist[i_star]
    kv_row = L * 2 * hp.Hkv * hp.D * 2
    trie_b = int(nh[i_star].sum()) * kv_row
    batch_b = R * (b if k_star > 0 else 1) * (t + k_star) * kv_row
    # batch beam search keeps b*(t+k) rows per request (prompt replicated, pending token
    # included: the paper's 21 = 3 x 7 counting); the trie keeps N rows
    res["kv_memory"] = dict(step_in_job=int(k_star), trie_bytes=trie_b, batch_bytes=batch_b,
                            trie_peak_bytes=int(nh.sum(axis=1).max()) * kv_row,
                            pool_bytes_allocated=int(2 * L * hp.Hkv * hp.D * 2 * (
                                hp.n_pages * 64 if hp.n_pages else R * hp.cap)),
                            ratio_batch_over_trie=round(batch_b / max(trie_b, 1), 3),
                            bound_b_ts_over_t_s_b_1=round(b * (t + k_star) / (t + k_star + b - 1), 3),
                            # the Fig. 3 analog: logical KV bytes before every timed
                            # step, trie (N rows) vs batch (b (t + k) rows per request), in MB
                            series=dict(step_in_job=[int(k) for k in k_hist],
                                        trie_MB=[round(float(nh[i].sum()) * kv_row / 1e6, 1)
                                                 for i in range(len(k_hist))],
                                        batch_MB=[round(R * (b if k > 0 else 1) * (t + k) * kv_row / 1e6, 1)
                                                  for k in k_hist]))
    res["execution"]["timed_job_steps"] = [int(k_hist[0]), int(k_hist[-1])]
    if args.series:
        res["series"] = run_series(hp, advance_to)
    if not args.no_e2e:
        res["e2e"] = run_e2e(hp, args, world)
    if args.model_context:  # last: it drives the trie with the model's own logits
        res["model_context"] = run_model_context(hp, args, world)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return res, dict(rank=rank, world=world)


def run_series(hp, advance_to):
    """--series: one whole job (s steps from k = 0) replayed with the instrumented graphs,
    synchronised per step: per-step attention (all L layers), beam-step and GC times
    (CUDA event nodes), the trie rows before each step (summed over requests) and batch
    beam search's b (t + k) rows -- the Fig. 4 (GC vs decoding pass) and
    tab:ablation (saved KV entries) experiments."""
    torch = hp.torch
    advance_to(0)
    torch.cuda.synchronize()
    out = dict(k=[], attn_ms=[], beam_ms=[], gc_ms=[], gc_ran=[], trie_rows=[], batch_rows=[],
               dead_rows=[], dead_tiles=[], tiles=[])
    for i in range(hp.s):
        k = hp.k
        rows = int(hp.st.n_nodes.sum().item()) if k > 0 else hp.R * hp.t
        # g > 1: generated rows no live beam sees (mask 0) and 64-row tiles made only of them
        # (the tiles a dead-tile skip could avoid; every depth keeps >= 1 live ancestor, so a
        # tile spanning >= 1 whole step of b <= 64 appended rows always holds a live row)
        dr = dt = nt = 0
        if k > 0:
            N = hp.st.n_nodes.cpu().numpy()
            msk = hp.st.beam_mask.cpu().numpy()
            for r in range(hp.R):
                gen = msk[r, hp.t: N[r]]
                dr += int(np.count_nonzero(gen == 0))
                for t0 in range(0, int(N[r]), 64):
                    nt += 1
                    if t0 >= hp.t and not np.any(msk[r, t0: min(t0 + 64, N[r])]):
                        dt += 1
        out["dead_rows"].append(dr)
        out["dead_tiles"].append(dt)
        out["tiles"].append(nt)
        key = hp.next_key()
        hp.replay(i % 2, timed=True)
        torch.cuda.synchronize()
        evs = hp.ev[(key, i % 2)]
        out["k"].append(k)
        out["attn_ms"].append(round(sum(e0.elapsed_time(e1) for e0, e1 in evs[:-2]), 4))
        out["beam_ms"].append(round(evs[-2][0].elapsed_time(evs[-2][1]), 4))
        out["gc_ms"].append(round(evs[-1][0].elapsed_time(evs[-1][1]) if key[1] else 0.0, 4))
        out["gc_ran"].append(bool(key[1]))
        out["trie_rows"].append(rows)
        out["batch_rows"].append(hp.R * (hp.b if k > 0 else 1) * (hp.t + k))
    tr, br = np.array(out["trie_rows"], float), np.array(out["batch_rows"], float)
    gc = np.array(out["gc_ms"])[np.array(out["gc_ran"])]
    pas = np.array(out["attn_ms"]) + np.array(out["beam_ms"])
    out["summary"] = dict(
        requests=hp.R, gc_interval=hp.g,
        saved_rows_per_request_mean=round(float((br - tr).mean()) / hp.R, 1),
        saved_rows_per_request_final=round(float(br[-1] - tr[-1]) / hp.R, 1),
        trie_over_batch_rows_mean=round(float((tr / br).mean()), 4),
        gc_ms_mean=round(float(gc.mean()), 4) if len(gc) else None,
        pass_ms_mean=round(float(pas.mean()), 4),
        gc_over_pass_max=round(float((np.array(out["gc_ms"]) / pas).max()), 4),
        dead_rows_mean=round(float(np.mean(out["dead_rows"])), 1),
        dead_tiles_total=int(np.sum(out["dead_tiles"])), tiles_total=int(np.sum(out["tiles"])),
        note="rows = KV entries (one per token per layer set); trie rows before each step, "
             "batch = b (t + k) per request (prompt replicated, P:42 counting)")
    return out


def run_model_context(hp, args, world):
    """--model-context: the same job with the random-init model around the hot path
    (paper_2502_00085_b200.model.ShapedModel: bf16 cuBLAS GEMMs for Q/K/V, O, MLP and LM
    head, the library's fused RoPE + append + trie attention per layer, the beam step on
    the model's own fp32 logits, GC), replayed as CUDA graphs.  Reports request-steps/s of
    the whole decode step and its breakdown (event nodes around every attention launch,
    the LM head, the beam step and GC; the rest is the layers' GEMMs and elementwise ops).
    SURVEY §8(d): "Report the breakdown: GEMM / attn / beam-step / prune"."""
    import torch

    from paper_2502_00085_b200.dist import gather_heads, heads_view
    from paper_2502_00085_b200.model import ShapedModel
    wl = hp.wl
    if "d" not in wl:
        raise SystemExit("--model-context: phi, llama or mistral-shard")
    m = ShapedModel(hp.L, wl["d"], wl["Hq"], wl["Hkv"], hp.D, wl["ffn"], hp.V, wl["theta"],
                    kappa=float(wl.get("kappa", 3.0)), q_heads=hp.Hq, kv_heads=hp.Hkv)
    st, L = hp.st, hp.L
    gather = None
    if hp.kv_shard and world > 1:
        def gather(o):
            if hp.eager:
                return heads_view(gather_heads(o.cpu())).to(o.device)
            dst = hp.gathered if o.shape[1] == hp.b else hp.gathered1
            return heads_view(gather_heads(o, dst))

    def step(var, events=None):
        if var == "first":
            st.reset()
        lg = m.step(st, hp.kp, hp.vp, gather=gather, events=None if events is None else events[:L + 1])
        if events is not None:
            events[L + 1][0].record()
        st.beam_step(lg, hp.sel_p, hp.sel_t, hp.sel_s)
        if events is not None:
            events[L + 1][1].record()
            events[L + 2][0].record()
        st.prune_compact(hp.kp, hp.vp)
        if events is not None:
            events[L + 2][1].record()

    ev = {v: [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
              for _ in range(L + 3)] for v in ("first", "steady")}
    step("first")
    step("steady")
    torch.cuda.synchronize()
    graphs = {}
    for var in ("first", "steady"):
        for timed in (False, True):
            if hp.eager:
                graphs[(var, timed)] = _Eager(lambda var=var, timed=timed: step(var, ev[var] if timed else None))
                continue
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                step(var, ev[var] if timed else None)
            graphs[(var, timed)] = gr
    k = [0]

    def replay(timed=False):
        var = "first" if k[0] == 0 else "steady"
        graphs[(var, timed)].replay()
        k[0] = (k[0] + 1) % hp.s
        return var
    for _ in range(args.warmup):
        replay()
    if args.steps < hp.s:
        while k[0] != (hp.s - args.steps) // 2:
            replay()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k_first = k[0]
    t0.record()
    for _ in range(args.steps):
        replay()
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device=hp.dev if not hp.eager else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    # breakdown over the same job steps of the next job (instrumented graphs, synced per step)
    while k[0] != k_first:
        replay()
    attn, lm, beam, gc, tot = [], [], [], [], []
    for _ in range(args.steps):
        a = torch.cuda.Event(enable_timing=True)
        z = torch.cuda.Event(enable_timing=True)
        a.record()
        var = replay(timed=True)
        z.record()
        torch.cuda.synchronize()
        e = ev[var]
        attn.append(sum(e[l][0].elapsed_time(e[l][1]) for l in range(L)))
        lm.append(e[L][0].elapsed_time(e[L][1]))
        beam.append(e[L + 1][0].elapsed_time(e[L + 1][1]))
        gc.append(e[L + 2][0].elapsed_time(e[L + 2][1]))
        tot.append(a.elapsed_time(z))
    assert st.status() == 0, f"device status bits {st.status():#x}"
    step_ms = ms / args.steps
    f = step_ms / float(np.mean(tot))  # scale the instrumented step to the plain one
    N = st.n_nodes.cpu().numpy()
    units = hp.R if hp.kv_shard else hp.R * world
    br = dict(attention=float(np.mean(attn)) * f, lm_head=float(np.mean(lm)) * f,
              beam_step=float(np.mean(beam)) * f, gc=float(np.mean(gc)) * f)
    br["layer_gemms_and_elementwise"] = step_ms - sum(br.values())
    return dict(value=round(units * args.steps / (ms * 1e-3), 2), unit="request-steps/s",
                ms_per_step=round(step_ms, 4), weights_GB=round(m.weight_bytes() / 1e9, 2),
                logit_scale=m.kappa,
                breakdown_ms_per_step={k_: round(v, 4) for k_, v in br.items()},
                trie_rows_end=int(N.sum()),
                model="random-init bf16 decoder of the workload's shape (cuBLAS GEMMs via torch; "
                      "prompt K/V rows synthetic); the library runs attention, beam step and GC",
                timing=f"{args.steps} CUDA-graph replays (job steps {k_first}..); breakdown from "
                       "event-instrumented replays of the same job steps, scaled to the plain step")


def run_e2e(hp, args, world):
    """Same steps, inputs copied from pinned host memory every step (copy stream,
    double-buffered), selections copied back to pinned host memory every step."""
    import torch
    import torch.distributed as dist
    host = {}
    for key, d in hp.inp.items():
        host[key] = dict(qkv=d["qkv"].cpu().pin_memory(), logits=d["logits"].cpu().pin_memory())
    out_host = [torch.empty(3, hp.R, hp.b, dtype=torch.int32).pin_memory() for _ in range(2)]
    compute = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    h2d = d2h = 0
    k_sim = hp.k

    def var_of(k):
        return "first" if k % hp.s == 0 else "steady"

    def prefetch(i, k):
        nonlocal h2d
        slot = i % 2
        var = var_of(k)
        with torch.cuda.stream(copy):
            copy.wait_event(ev_free[slot])
            hp.inp[(var, slot)]["qkv"].copy_(host[(var, slot)]["qkv"], non_blocking=True)
            hp.inp[(var, slot)]["logits"].view(-1).copy_(host[(var, slot)]["logits"].view(-1), non_blocking=True)
            ev_in[slot].record(copy)
        h2d += host[(var, slot)]["qkv"].numel() * 2 + host[(var, slot)]["logits"].numel() * 4

    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for e in ev_free:
        e.record(compute)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(compute)
    copy.wait_event(t0)
    prefetch(0, k_sim)
    for i in range(args.steps):
        slot = i % 2
        compute.wait_event(ev_in[slot])
        hp.replay(slot)
        ev_free[slot].record(compute)
        if i + 1 < args.steps:
            prefetch(i + 1, k_sim + i + 1)
        oh = out_host[slot]
        oh[0].copy_(hp.sel_p, non_blocking=True)
        oh[1].copy_(hp.sel_t, non_blocking=True)
        oh[2].copy_(hp.sel_s.view(torch.int32), non_blocking=True)
        d2h += 3 * hp.R * hp.b * 4
    t1.record(compute)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], device=hp.dev if os.environ.get("BENCH_DIST_BACKEND", "nccl") == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    units = hp.R if hp.kv_shard else hp.R * world
    return {"value": round(units * args.steps / (ms * 1e-3), 2), "unit": "request-steps/s",
            "h2d_bytes_per_step": int(h2d // args.steps), "d2h_bytes_per_step": int(d2h // args.steps),
            "ms_per_step": round(ms / args.steps, 4),
            "path": "C ABI via the binding; pinned host -> device copies on a side stream, "
                    "double-buffered; selections device -> pinned host every step"}


def _traffic(workload, R, b):
    """dram bytes per attention launch from the committed ncu --set full summary, when it
    was captured on this exact workload (same requests per GPU and beam width)."""
    p = os.path.join(ROOT, "profiles", "ncu_attn_summary.json")
    if os.path.exists(p):
        try:
            e = json.load(open(p)).get(workload, {})
            if e.get("requests") == R and e.get("beam") == b:
                return e.get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


# ------------------------------------------------------------------------------------------
# CPU oracle timing (the cpu_baseline leg and --impl reference): the oracle as it stands,
# on the host cores of this box, over independent requests (the natural DP axis, SURVEY
# §8(d)): one worker process per core, each one request, numpy fp64 with ONE BLAS thread.
def cpu_info():
    """nproc, usable cores, lscpu model and sockets of this host."""
    info = {"nproc": os.cpu_count(), "usable_cores": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() == "Model name":
                info["model"] = v.strip()
            elif k.strip() == "Socket(s)":
                info["sockets"] = v.strip()
    except Exception:
        pass
    return info


def _oracle_request(wl, req):
    """One request of the workload at mid-job, built by the oracle itself: prompt (synth,
    the bench's recipe), then k_mid = s/2 steps of the oracle's beam step over seeded
    N(0, 3^2) logits (the bench's logit scale) with the trie update and GC of Alg. 2.
    Q / K / V of the step are N(0, 1) (the bench's inputs); K / V [Hkv][N][D] stand for
    one layer's pool, re-used by all L layers (each layer still runs attn_ref in full)."""
    import synth
    from oracle.kernels_ref import beam_step_ref
    from oracle.trie import Trie, garbage_collect
    t, b, V, s = wl["t"], wl["b"], wl["V"], wl["s"]
    prompts, _ = synth.prompts(10_000 + req, 1, t, V)
    T = Trie(prompts[0])
    for k in range(s // 2):
        lg = synth.normal(5_000 + req, k, (len(T.leaves), V)) * 3.0
        par, tok, cs, _, _ = beam_step_ref(lg, T.scores, b)
        T.update_trie([(float(c), int(v), int(j)) for c, v, j in zip(cs, tok, par)])
        garbage_collect(T)
    Hq, Hkv, D = wl["Hq"], wl["Hkv"], wl["D"]
    return dict(T=T, q=synth.normal(6_000 + req, 1, (b, Hq, D)),
                K=synth.normal(6_000 + req, 2, (Hkv, T.N, D)),
                Vv=synth.normal(6_000 + req, 3, (Hkv, T.N, D)),
                logits=synth.normal(6_000 + req, 4, (b, V)) * 3.0)


def _oracle_request_step(st, wl):
    """One request-step on the CPU oracle: L x attn_ref (a-3, every layer computed) +
    beam_step_ref (a-4) + trie append (a-5) + GC mark / prune / compact (a-6) on a copy
    (so every step starts from the same mid-job state)."""
    import copy
    from oracle.kernels_ref import attn_ref, beam_step_ref
    from oracle.trie import garbage_collect
    T = st["T"]
    for _ in range(wl["L"]):
        attn_ref(st["q"], st["K"], st["Vv"], T, window=wl["W"])
    par, tok, cs, _, _ = beam_step_ref(st["logits"], T.scores, wl["b"])
    Tc = copy.deepcopy(T)
    Tc.update_trie([(float(c), int(v), int(j)) for c, v, j in zip(cs, tok, par)])
    garbage_collect(Tc)


def _oracle_worker(conn, wl, req):
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):
        st = _oracle_request(wl, req)
        conn.send(("ready", st["T"].N))
        while conn.recv() is not None:
            a = time.perf_counter()
            _oracle_request_step(st, wl)
            conn.send(time.perf_counter() - a)


def cpu_oracle_run(wl, steps, warmup, workers=None, budget_s=None):
    """Time `steps` parallel request-steps (after `warmup`) of `workers` independent
    requests (default: every usable core, at most 128), one process each, numpy with one
    BLAS thread.  Returns (request-steps/s, dict of details).  Wall time per step is the
    host clock around one request-step of every worker; `budget_s` stops early."""
    import multiprocessing as mp
    P = workers or min(len(os.sched_getaffinity(0)), 128)
    env_keep = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in env_keep:
        os.environ[k] = "1"
    ctx = mp.get_context("spawn")
    procs, conns = [], []
    try:
        for i in range(P):
            a, c = ctx.Pipe()
            p = ctx.Process(target=_oracle_worker, args=(c, wl, i), daemon=True)
            p.start()
            procs.append(p)
            conns.append(a)
        Ns = [c.recv()[1] for c in conns]
        walls, per_req = [], []
        t_start = None
        for i in range(warmup + steps):
            a = time.perf_counter()
            for c in conns:
                c.send(1)
            dts = [c.recv() for c in conns]
            w = time.perf_counter() - a
            if i >= warmup:
                if t_start is None:
                    t_start = a
                walls.append(w)
                per_req.extend(dts)
                if budget_s is not None and time.perf_counter() - t_start > budget_s:
                    break
        for c in conns:
            c.send(None)
    finally:
        for p in procs:
            p.join(timeout=5)
            if p.is_alive():
                p.terminate()
        for k, v in env_keep.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    wall = float(np.sum(walls))
    return P * len(walls) / wall, dict(
        workers=P, steps=len(walls), wall_s=round(wall, 3), ms_per_step=round(wall / len(walls) * 1e3, 6),
        per_request_step_s=round(float(np.mean(per_req)), 4), trie_rows_mean=round(float(np.mean(Ns)), 1))


def _oracle_sample_text(wl, d):
    return (f"{d['workers']} independent requests in parallel (one process per core, numpy fp64, "
            f"1 BLAS thread each), {d['steps']} timed steps; each worker step = one request-step at "
            f"step {wl['s'] // 2} of its job (oracle-built trie, {d['trie_rows_mean']} rows mean): "
            f"attn_ref on all {wl['L']} layers (one layer's K/V re-used) + beam_step_ref over "
            f"b x V + append + GC; host wall clock per step")


def cpu_baseline(wl, budget_s=12.0):
    v, d = cpu_oracle_run(wl, steps=64, warmup=1, budget_s=budget_s)
    return {"value": round(v, 4), "unit": "request-steps/s", "cores": d["workers"], "kind": "oracle",
            "sample": _oracle_sample_text(wl, d), "host": cpu_info(), **d}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands on this box's host cores, on the GPU
    arm's workload, metric, unit and config; K timed steps after W warm-up steps, each
    step a request-step of every worker (rank 0 only; other ranks exit without work)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    wl = _workload(args)
    v, d = cpu_oracle_run(wl, steps=args.steps, warmup=args.warmup)
    res = dict(metric=METRIC, value=round(v, 4), unit="request-steps/s", n_gpus=world, steps=d["steps"],
               warmup=args.warmup, ms_per_step=d["ms_per_step"], higher_is_better=True,
               scaling=_scaling(wl), vs_baseline=None, dtype="f64", data="synthetic", impl="reference",
               config=bench_config(wl, world),
               cpu_baseline=dict(value=round(v, 4), unit="request-steps/s", cores=d["workers"], kind="oracle",
                                 sample=_oracle_sample_text(wl, d), host=cpu_info(), **d),
               e2e=dict(value=round(v, 4), unit="request-steps/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    return res


def run_oracle_units(args):
    """--impl reference --units: SURVEY §8(d)'s per-unit CPU oracle timings on this host
    (1 thread each): configs[0] full decodes (trie and batch, seconds), attn_ref per
    (request, layer) at every bench shape, beam_step_ref at each V, GC."""
    import copy

    from threadpoolctl import threadpool_limits

    import synth
    from oracle.decode import batch_beam_search, trie_beam_search
    from oracle.kernels_ref import attn_ref, beam_step_ref, build_tries
    from oracle.model import Model, ModelConfig
    from oracle.trie import garbage_collect
    out = dict(kind="oracle per-unit timings, 1 thread", host=cpu_info(), units=[])

    def timeit(fn, reps):
        ts = []
        for _ in range(reps):
            a = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - a)
        return float(np.median(ts))

    with threadpool_limits(limits=1):
        # configs[0]: tiny 2-layer MHA, prompt 8, b=3, 16 steps (fp64 oracle, seconds)
        seed = 0
        m = Model(synth.tiny_weights(seed, 2, 64, 4, 4, 16, 256, 256), ModelConfig())
        prompts, _ = synth.prompts(seed, 1, 8, 256)
        p0 = [int(x) for x in prompts[0]]
        out["units"].append(dict(unit="configs[0] full decode, trie (Alg. 2)", seconds=round(
            timeit(lambda: trie_beam_search(m, p0, 3, 16, g=1), 3), 4)))
        out["units"].append(dict(unit="configs[0] full decode, batch (Alg. 1)", seconds=round(
            timeit(lambda: batch_beam_search(m, p0, 3, 16), 3), 4)))
        shapes = [("phi", {}), ("llama", {}), ("mistral-shard", {}), ("sweep", {"b": 16})]
        for name, over in shapes:
            wl = dict(WORKLOADS[name], **over)
            t, b, V, s = wl["t"], wl["b"], wl["V"], wl["s"]
            pr, ln = synth.prompts(1, 1, t, V)
            sels = [(p_[None], q_[None]) for p_, q_ in synth.selections(3, s // 2, b, V, 0.5)]
            T = build_tries(pr, ln, sels, b, g=1)[0]
            q = synth.normal(4, 1, (b, wl["Hq"], wl["D"]))
            K = synth.normal(4, 2, (wl["Hkv"], T.N, wl["D"]))
            Vv = synth.normal(4, 3, (wl["Hkv"], T.N, wl["D"]))
            lg = synth.normal(4, 4, (b, V)) * 3.0
            sc = np.zeros(b)
            a = timeit(lambda: attn_ref(q, K, Vv, T, window=wl["W"]), 2)
            bs = timeit(lambda: beam_step_ref(lg, sc, b), 2)
            par, tok, cs, _, _ = beam_step_ref(lg, sc, b)

            def gc_unit():
                Tc = copy.deepcopy(T)
                Tc.update_trie([(float(c), int(v), int(j)) for c, v, j in zip(cs, tok, par)])
                garbage_collect(Tc)
            gcs = timeit(gc_unit, 3)
            out["units"].append(dict(
                unit=f"{wl['name']} b={b}: request at step {s // 2} (dial rho=0.5, N={T.N})",
                attn_ref_per_request_layer_s=round(a, 4), beam_step_ref_s=round(bs, 4),
                append_gc_s=round(gcs, 5), request_step_all_layers_s=round(wl["L"] * a + bs + gcs, 3)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="phi", choices=sorted(WORKLOADS))
    ap.add_argument("--beam", type=int, default=0)
    ap.add_argument("--requests", type=int, default=0)
    ap.add_argument("--gc-interval", type=int, default=1,
                    help="Alg. 2's GC interval g (1 = every step, the hot path; 0 = never)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "batch"],
                    help="ours | reference (CPU oracle) | batch (GPU batch beam search, NEXT-2)")
    ap.add_argument("--eos-frac", type=float, default=0.0,
                    help="NEXT-3 experiment: EOS id 0 finishes this fraction of the requests early")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--series", action="store_true",
                    help="NEXT-1 experiments: one whole instrumented job, per-step times and rows")
    ap.add_argument("--model-context", action="store_true",
                    help="also time the step inside a random-init model of the workload's shape")
    ap.add_argument("--paged", type=float, default=0.5,
                    help="NEXT-2: paged KV pools sized prompt + f x the no-GC generated pages "
                         "(0: dense pools sized for the no-GC worst case)")
    ap.add_argument("--prompt-len", type=int, default=0)
    ap.add_argument("--new-tokens", type=int, default=0)
    ap.add_argument("--logit-scale", type=float, default=0.0,
                    help="scale of the synthetic N(0, 1) logits (the convergence knob kappa; default 3)")
    ap.add_argument("--units", action="store_true",
                    help="with --impl reference: SURVEY 8(d) per-unit CPU oracle timings (1 thread)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        res = run_oracle_units(args) if args.units else run_reference(args)
        if res is not None:
            print(json.dumps(res))
        return
    if args.impl == "batch":
        print(json.dumps(run_batch(args)))
        return
    res, ctx = run_gpu(args)
    if ctx["rank"] == 0:
        if not args.no_cpu_baseline and ctx["world"] == 1:
            res["cpu_baseline"] = cpu_baseline(_workload(args))
        print(json.dumps(res))


if __name__ == "__main__":
    main()
