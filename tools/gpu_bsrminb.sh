#!/bin/bash
# BSR min-CTAs-per-SM A/B: square row kernels (TMG_BSR_MINB) x transfer kernels
# (TMG_BSR_XFER_MINB), builds under lib/ab/ selected through TMG_LIB, made with
#   nvcc <_build.NVCC_FLAGS> -DTMG_BSR_MINB=a -DTMG_BSR_XFER_MINB=b -o paper_2001_01655_b200/lib/ab/libtopomg_sqa_xfb.so paper_2001_01655_b200/csrc/tmg_abi.cu
mkdir -p gpurun_out
for v in sq4_xf4 sq4_xf6 sq1_xf6; do
  export TMG_LIB=$PWD/paper_2001_01655_b200/lib/ab/libtopomg_$v.so
  timeout 300 python tools/iter_breakdown.py --config 1 --legs amg > gpurun_out/bm_c1_$v.log 2>&1
  timeout 400 python tools/iter_breakdown.py --config 2 > gpurun_out/bm_c2_$v.log 2>&1
  timeout 600 python tools/iter_breakdown.py --config 4 > gpurun_out/bm_c4_$v.log 2>&1
done
echo done
