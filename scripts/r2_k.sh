#!/bin/bash
TAG=${1:-r2k}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for wl in phi llama; do
  for pg in 0 0.5; do
    timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --paged $pg > gpurun_out/${TAG}_${wl}_p$pg.json 2>gpurun_out/${TAG}_${wl}_p$pg.err
  done
done
tail -n 3 gpurun_out/${TAG}_pytest.log
