#!/bin/bash
# A/B round trip: parity suite, then per-level iteration breakdowns.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
TMG_SA_FACTORED=0 timeout 300 python tools/iter_breakdown.py --config 1 > gpurun_out/brk_c1_stored.log 2>&1
timeout 300 python tools/iter_breakdown.py --config 1 > gpurun_out/brk_c1.log 2>&1
for c in ${CONFIGS:-2 3 4}; do
  timeout 600 python tools/iter_breakdown.py --config $c --iters 200 > gpurun_out/brk_c$c.log 2>&1
done
echo done
