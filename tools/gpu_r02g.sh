#!/bin/bash
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "not checkpoints" ) 2>&1 | tail -15 > gpurun_out/pytest_gpu_nockpt.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_sens3.log 2>&1
TMG_SENS_GATHER=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_sens_gather.log 2>&1
echo done
