#!/bin/bash
# final insurance run of HEAD: GPU tests, smoke, the driver's default bench command
TAG=${1:-r2f7}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2>gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2>gpurun_out/${TAG}_ref.err
tail -n 2 gpurun_out/${TAG}_pytest.log gpurun_out/${TAG}_smoke.log; cat gpurun_out/${TAG}_bench.json | head -c 400
