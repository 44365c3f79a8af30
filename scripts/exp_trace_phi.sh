TRIE_BUILD_DEFINES="TRIE_ATTN_TRACE=1" python -m paper_2502_00085_b200.build --force >/dev/null
python scripts/attn_trace.py --workload phi --step 30 > gpurun_out/trace41_phi.txt 2>&1
python scripts/attn_trace.py --workload llama --step 131 > gpurun_out/trace41_llama.txt 2>&1
python -m paper_2502_00085_b200.build --force >/dev/null
python - > gpurun_out/readbw41.txt 2>&1 <<'PY'
import torch
x = torch.empty(2**31, dtype=torch.bfloat16, device="cuda").normal_()
for _ in range(3): x.sum()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): x.sum()
e1.record(); torch.cuda.synchronize()
print("torch sum read GB/s", 10 * x.numel() * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
y = torch.empty_like(x)
e0.record()
for _ in range(10): y.copy_(x)
e1.record(); torch.cuda.synchronize()
print("copy (r+w) GB/s", 10 * x.numel() * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
PY
