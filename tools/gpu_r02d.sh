#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tests/diagnostics/c1_gmg_gap2.py > gpurun_out/c1_gmg_gap2.log 2>&1
echo done
