#!/bin/bash
# x-only last Chebyshev step A/B + full parity suite
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ) 2>&1 | tail -30 > gpurun_out/pytest_gpu_all.log
for x in 1 0; do
  echo "=== TMG_CHEB_XONLY=$x" >> gpurun_out/xonly_ab.txt
  TMG_CHEB_XONLY=$x timeout 600 python tools/iter_breakdown.py --config 4 2>&1 | head -3 >> gpurun_out/xonly_ab.txt
  TMG_CHEB_XONLY=$x timeout 600 python tools/iter_breakdown.py --config 3 2>&1 | head -3 >> gpurun_out/xonly_ab.txt
done
echo done
