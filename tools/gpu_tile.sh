#!/bin/bash
# A/B of tile shapes: libtopomg_b200{,_a,_b}.so built with different -DTMG_F?_B? flags
mkdir -p gpurun_out
for v in "" _a _b; do
  TMG_LIB=$PWD/paper_2001_01655_b200/lib/libtopomg_b200$v.so timeout 300 python tools/iter_breakdown.py --config ${C:-1} > gpurun_out/tile$v.txt 2>&1
done
