#!/bin/bash
# ncu --set full (with SASS-level stall sampling) of the level-0 Chebyshev step inside an eager PCG iteration of config 4
mkdir -p gpurun_out
export TMG_PCG_EAGER=1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:k_chebILi3ENS_6FineOp -s 2 --launch-count 1 \
   -o gpurun_out/ncu_cheb3d -f python tools/profile_case.py --config 4 --iters 3 --reps 1 > gpurun_out/ncu_cheb3d.log 2>&1
echo done
