#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/coarse_accuracy.txt
for m in chol gj; do TMG_COARSE=$m timeout 600 python tests/diagnostics/coarse_accuracy.py >> gpurun_out/coarse_accuracy.txt 2>&1; done
echo done
