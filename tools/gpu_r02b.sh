#!/bin/bash
# Round-2 GPU trip B: full parity suite (no -x), config-1 GMG checkpoints with both coarse inverses,
# FP64 peak, ncu --set full of the config-4 level-0 kernels.
mkdir -p gpurun_out
tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ) 2>&1 | tail -60 > gpurun_out/pytest_gpu_all.log
TMG_COARSE=gj timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -s -k "config1_checkpoints" 2>&1 | grep -E "k=|passed|failed|Error" > gpurun_out/c1_ckpt_gj.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -s -k "config1_checkpoints" 2>&1 | grep -E "k=|passed|failed|Error" > gpurun_out/c1_ckpt_chol.log
export TMG_PCG_EAGER=1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:k_chebILi3ENS_6FineOp -s 2 --launch-count 1 \
   -o gpurun_out/ncu_cheb3d -f python tools/profile_case.py --config 4 --iters 3 --reps 1 > gpurun_out/ncu_cheb3d.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:k_residualILi3ENS_6FineOp -s 1 --launch-count 1 \
   -o gpurun_out/ncu_res3d -f python tools/profile_case.py --config 4 --iters 3 --reps 1 > gpurun_out/ncu_res3d.log 2>&1
echo done
