#!/bin/bash
mkdir -p gpurun_out
for c in ${CONFIGS:-3 4}; do
  for v in _m2 _m3 _m4; do
    TMG_LIB=$PWD/paper_2001_01655_b200/lib/libtopomg_b200$v.so timeout 900 python tools/roofline_table.py --config $c --reps 20 > gpurun_out/roofline${v}_c$c.txt 2>&1
  done
done
echo done
