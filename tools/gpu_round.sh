#!/bin/bash
# One GPU round trip (gpurun -- 'bash tools/gpu_round.sh'): parity suite with the
# checkpoint table, smoke, default bench, per-level breakdown of configs 3 and 4.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.log
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s ) 2>&1 | grep -E "k=|passed|failed|Error|real" > gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
( time timeout 900 python bench.py ) > gpurun_out/bench.log 2>&1
for c in ${CONFIGS:-4 3}; do timeout 600 python tools/iter_breakdown.py --config $c > gpurun_out/iter_breakdown_c$c.txt 2>&1; done
echo done
