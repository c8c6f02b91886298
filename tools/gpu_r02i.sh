#!/bin/bash
mkdir -p gpurun_out
( timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_amg.py tests/test_gpu_krylov.py tests/test_gpu_sor.py tests/test_gpu_host_entry.py -m gpu -q -p no:cacheprovider ) 2>&1 | tail -40 > gpurun_out/pytest_gpu_small.log
for m in chol gj; do
  echo "=== TMG_COARSE=$m" >> gpurun_out/pytest_gpu_small.log
  TMG_COARSE=$m TMG_VERBOSE=1 timeout 600 python tools/profile_case.py --config 1 --iters 5 --legs gmg 2>&1 | grep -E "coarse|setup_ms" >> gpurun_out/pytest_gpu_small.log
  TMG_COARSE=$m timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3 >> gpurun_out/pytest_gpu_small.log
done
echo done
