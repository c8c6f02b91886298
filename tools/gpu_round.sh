#!/bin/bash
# One GPU round trip: parity suite, per-leg timings of a config, short bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-1}; do
  TMG_VERBOSE=1 timeout 600 python tools/profile_case.py --config $c --iters ${ITERS:-3000} > gpurun_out/profile_c$c.log 2>&1
done
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
echo done
