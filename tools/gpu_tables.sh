#!/bin/bash
mkdir -p gpurun_out
for c in ${CONFIGS:-1 2 3 4}; do
  timeout 900 python tools/roofline_table.py --config $c > gpurun_out/roofline_c$c.txt 2>&1
done
timeout 600 python tools/sor_timing.py --config 1 > gpurun_out/sor_c1.txt 2>&1
echo done
