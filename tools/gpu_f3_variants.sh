#!/bin/bash
# A/B of the 3D level-0 operator builds (TMG_LIB selects the library): 3D parity subset + config-4 timings.
mkdir -p gpurun_out
for v in ${VARIANTS:-topomg_b200 tmg_ty12 tmg_ty6 tmg_tma}; do
  export TMG_LIB=$PWD/paper_2001_01655_b200/lib/lib$v.so
  [ -f "$TMG_LIB" ] || { echo "missing $TMG_LIB"; continue; }
  echo "=== $v" > gpurun_out/f3_$v.log
  timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "operator or vcycle or hybrid_matches or linear_and_symmetric or 3d or gmg" 2>&1 | tail -5 >> gpurun_out/f3_$v.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke_3d()" >> gpurun_out/f3_$v.log 2>&1
  timeout 600 python tools/iter_breakdown.py --config 4 2>&1 | head -4 >> gpurun_out/f3_$v.log
  timeout 600 python tools/iter_breakdown.py --config 3 2>&1 | head -3 >> gpurun_out/f3_$v.log
done
echo done
