#!/bin/bash
# parity suite with the regenerated fixtures, default bench, config 3/4 iteration breakdown
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s ) 2>&1 | grep -E "k=|passed|failed|Error|real" > gpurun_out/pytest_gpu_all.log
timeout 600 python tools/iter_breakdown.py --config 4 > gpurun_out/iter_breakdown_c4.txt 2>&1
timeout 600 python tools/iter_breakdown.py --config 3 > gpurun_out/iter_breakdown_c3.txt 2>&1
( time timeout 900 python bench.py ) > gpurun_out/bench.log 2>&1
echo done
