#!/bin/bash
mkdir -p gpurun_out
export TMG_PCG_EAGER=1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:k_residualILi3ENS_6FineOp --launch-count 1 \
   -o gpurun_out/ncu_res3d -f python tools/profile_case.py --config 3 --iters 3 --reps 1 > gpurun_out/ncu3.log 2>&1
echo done
