#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sor.py -q -x -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_sor.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
echo done
