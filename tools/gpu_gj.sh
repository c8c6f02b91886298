#!/bin/bash
# Coarse Gauss-Jordan pass: parity suite, GMG setup phases, launch list of the
# GMG leg, one --set full capture per Gauss-Jordan kernel, bench line.
mkdir -p gpurun_out
R=${ROUND:-r01}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/gj_pytest.log
TMG_VERBOSE=1 timeout 300 python tools/profile_case.py --config 1 --iters 20 --reps 3 --legs gmg > gpurun_out/gj_setup.log 2>&1
TMG_DENSE_MMA=0 TMG_VERBOSE=1 timeout 300 python tools/profile_case.py --config 1 --iters 20 --reps 3 --legs gmg > gpurun_out/gj_setup_nomma.log 2>&1
export TMG_PCG_EAGER=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_gmg_$R.csv python tools/profile_case.py --config 1 --iters 20 --reps 1 --legs gmg \
  > gpurun_out/ncu_gmg.log 2>&1
for k in k_gj_update_mma k_gj_panels k_gj_pivot; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 40 -c 1 -o gpurun_out/full_${k}_$R \
    python tools/profile_case.py --config 1 --iters 2 --reps 1 --legs gmg > gpurun_out/full_$k.log 2>&1
done
unset TMG_PCG_EAGER
timeout 900 python bench.py > gpurun_out/gj_bench.log 2>&1
echo done
