#!/bin/bash
# Iteration breakdowns only (A/B switches via env), no parity suite.
mkdir -p gpurun_out
TMG_SA_FACTORED=0 timeout 300 python tools/iter_breakdown.py --config ${C:-1} --legs ${LEGS:-gmg,amg} > gpurun_out/brk_stored.log 2>&1
timeout 300 python tools/iter_breakdown.py --config ${C:-1} --legs ${LEGS:-gmg,amg} > gpurun_out/brk.log 2>&1
echo done
