#!/bin/bash
# Round profiling pass: bench line, ncu launch list of the bench command (eager PCG
# so the graph's kernels are visible), one --set full capture per key kernel.
mkdir -p gpurun_out
R=${ROUND:-r01}
timeout 900 python bench.py > gpurun_out/bench_$R.log 2>&1
export TMG_PCG_EAGER=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_C:-6000} --csv \
  --log-file gpurun_out/launches_bench_$R.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --iters-cap 50 --e2e-steps 1 \
  > gpurun_out/ncu_bench_$R.log 2>&1
for spec in "fine_jacobi:_ZN3tmg8k_jacobiILi2ENS_6FineOpILi2EEELb0EEEvT0_PKdS5_S5_S5_PdNS_3RedE:gmg:4" \
            "fine_jacobi_dot:_ZN3tmg8k_jacobiILi2ENS_6FineOpILi2EEELb1EEEvT0_PKdS5_S5_S5_PdNS_3RedE:gmg:2" \
            "bsr_jacobi:_ZN3tmg12k_bsr_jacobiILi3ELb0EEEvNS_7BsrViewIXT_EXT_EEEPKdS4_S4_S4_PdNS_3RedE:amg:0" \
            "gemv:_ZN3tmg11k_gemv_rowsEPKdxS1_Pd:gmg:2"; do
  IFS=: read name kern leg skip <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "$kern" -s $skip -c 1 -o gpurun_out/${name}_$R \
    python tools/profile_case.py --config 1 --iters 5 --reps 1 --legs $leg > gpurun_out/full_${name}.log 2>&1
done
echo done
