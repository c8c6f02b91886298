#!/bin/bash
# same-box A/B of libtopomg_b200_before.so (previous build) vs the current build
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/pytest_gpu.log
for v in _before ""; do
  for c in ${CONFIGS:-1 3 4}; do
    TMG_LIB=$PWD/paper_2001_01655_b200/lib/libtopomg_b200$v.so timeout 300 python tools/iter_breakdown.py --config $c --iters 100 > gpurun_out/ab$c$v.txt 2>&1
  done
done
echo done
