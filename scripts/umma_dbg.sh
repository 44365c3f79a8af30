#!/bin/bash
# tcgen05 attention experiments (sweep shape, R=16): per-launch time by softmax layout (SW)
# and with the softmax math (dbg=1) or the MMAs (dbg=2) removed.  Timing only.
OUT=${1:-gpurun_out/dbg.txt}
for b in 16 32; do for sw in ${SWS:-2 4}; do for d in ${DBGS:-0 2}; do
echo "b=$b sw=$sw dbg=$d $(TRIE_UMMA_SW=$sw TRIE_UMMA_DBG=$d timeout 120 python scripts/attn_only.py --workload sweep --beam $b 2>&1 | tail -1)"
done; done; done > $OUT 2>&1
