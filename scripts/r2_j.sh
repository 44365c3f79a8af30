#!/bin/bash
# paged pools (NEXT-2) parity + tcgen05 regression A/B (alt builds via TRIE_LIB)
TAG=${1:-r2j}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 1200 python -m pytest tests/test_gpu_integer_path.py tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
  for v in cur old qbar; do
    case $v in cur) L="";; old) L=$PWD/alt/lib_oldumma.so;; qbar) L=$PWD/alt/lib_qbar.so;; esac
    TRIE_LIB=$L timeout 600 python bench.py --workload sweep --beam 16 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_${v}_sw16_$rep.json
    TRIE_LIB=$L timeout 600 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_${v}_mis_$rep.json
  done
done
tail -n 3 gpurun_out/${TAG}_pytest.log
