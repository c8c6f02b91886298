#!/bin/bash
# Gauss-Jordan A/B: parity suite on both update paths, setup timings of both.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/gj2_pytest.log
TMG_DENSE_MMA=0 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/gj2_pytest_nomma.log
for rep in 1 2; do
TMG_VERBOSE=1 timeout 300 python tools/profile_case.py --config 1 --iters 20 --reps 3 --legs gmg > gpurun_out/gj2_setup_$rep.log 2>&1
TMG_DENSE_MMA=0 TMG_VERBOSE=1 timeout 300 python tools/profile_case.py --config 1 --iters 20 --reps 3 --legs gmg > gpurun_out/gj2_setup_nomma_$rep.log 2>&1
done
export TMG_PCG_EAGER=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gj_update -s 40 -c 1 -o gpurun_out/full_k_gj_update_mma2 \
    python tools/profile_case.py --config 1 --iters 2 --reps 1 --legs gmg > gpurun_out/full_mma2.log 2>&1
TMG_DENSE_MMA=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gj_update -s 40 -c 1 -o gpurun_out/full_k_gj_update_scalar \
    python tools/profile_case.py --config 1 --iters 2 --reps 1 --legs gmg > gpurun_out/full_scalar.log 2>&1
echo done
