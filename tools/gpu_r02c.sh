#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tests/diagnostics/c1_gmg_gap.py 1 0 > gpurun_out/c1_gmg_gap.log 2>&1
timeout 900 python tests/diagnostics/c1_gmg_gap.py 3 0 > gpurun_out/c3_gmg_gap.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -s -k "checkpoints" 2>&1 | grep -E "k=|passed|failed|Error" > gpurun_out/ckpt_all.log
echo done
