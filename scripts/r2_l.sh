#!/bin/bash
TAG=${1:-r2l}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
bash scripts/sanitize.sh $TAG
tail -n 3 gpurun_out/${TAG}_pytest.log
