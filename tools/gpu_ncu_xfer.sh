#!/bin/bash
# --set full of the SA level-0 transfer kernels of config 1 (AMG leg) after the
# occupancy bounds: k_bsr_apply<2,3> (prolongation), k_bsr_restrict<3,2>.
mkdir -p gpurun_out
export TMG_PCG_EAGER=1
for k in k_bsr_applyILi2ELi3E k_bsr_restrictILi3ELi2E; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"$k" -s 2 -c 1 -o gpurun_out/full_${k}_r01 \
    python tools/profile_case.py --config 1 --iters 3 --reps 1 --legs amg > gpurun_out/full_$k.log 2>&1
done
echo done
