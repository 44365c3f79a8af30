#!/bin/bash
# beam step: unrolled rank counting (default) vs HEAD (alt_src/, git archive, not committed)
# vs rank counting up to 512 keys (TRIE_RANK_MAX=512): parity + microbench + llama
TAG=${1:-r2b1}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
(cd alt_src && TRIE_BUILD_OUT=/tmp/alt_b1.so python -m paper_2502_00085_b200.build --force >/dev/null)
TRIE_BUILD_OUT=/tmp/rank512.so TRIE_BUILD_DEFINES="TRIE_RANK_MAX=512" python -m paper_2502_00085_b200.build --force >/dev/null
timeout 900 python -m pytest tests/test_gpu_beam_step.py tests/test_gpu_integer_path.py tests/test_gpu_e2e_tiny.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
TRIE_LIB=/tmp/rank512.so timeout 900 python -m pytest tests/test_gpu_beam_step.py -m gpu -q -x > gpurun_out/${TAG}_pytest512.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest512.log
for rep in 1 2; do
  timeout 300 python scripts/bench_beam_step.py > gpurun_out/${TAG}_beam_default_$rep.json 2>&1
  TRIE_LIB=/tmp/alt_b1.so timeout 300 python scripts/bench_beam_step.py > gpurun_out/${TAG}_beam_alt_$rep.json 2>&1
  TRIE_LIB=/tmp/rank512.so timeout 300 python scripts/bench_beam_step.py > gpurun_out/${TAG}_beam_r512_$rep.json 2>&1
done
tail -2 gpurun_out/${TAG}_pytest.log gpurun_out/${TAG}_pytest512.log
for f in gpurun_out/${TAG}_beam_*.json; do echo $f; cat $f; done
