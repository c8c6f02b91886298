#!/bin/bash
# Round-2 profiling pass (one GPU): bench lines of both arms, the ncu launch list of the
# bench command (eager PCG so the graph's kernels are visible), one --set full capture
# per key kernel, roofline tables, setup timings.
mkdir -p gpurun_out
R=r02
( time timeout 900 python bench.py ) > gpurun_out/bench_$R.log 2>&1
( time timeout 1500 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup 1 ) > gpurun_out/bench_ref_$R.log 2>&1
for c in 1 2 3 4; do timeout 600 python tools/roofline_table.py --config $c > gpurun_out/roofline_c$c.txt 2>&1; done
timeout 900 python tools/config_table.py > gpurun_out/configs_$R.txt 2>&1
for m in chol gj; do
  echo "=== TMG_COARSE=$m" >> gpurun_out/setup_$R.txt
  TMG_COARSE=$m TMG_VERBOSE=1 timeout 600 python tools/profile_case.py --config 1 --iters 5 --legs gmg >> gpurun_out/setup_$R.txt 2>&1
done
TMG_VERBOSE=1 timeout 600 python tools/profile_case.py --config 4 --iters 5 >> gpurun_out/setup_$R.txt 2>&1
export TMG_PCG_EAGER=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_bench_$R.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 \
  > gpurun_out/ncu_bench_$R.log 2>&1
cap() {  # name, mangled-kernel regex, skip, config, legs
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:$2" -s $3 -c 1 -o gpurun_out/full_$1_$R -f \
    python tools/profile_case.py --config $4 --iters 3 --reps 1 ${5:+--legs $5} > gpurun_out/full_$1.log 2>&1
  digest full_$1_$R
}
digest() {  # keep the text pages, drop the (tens of MB) report: gpurun_out/ is capped at 64 MiB
  ncu -i gpurun_out/$1.ncu-rep --page details > gpurun_out/$1.details.txt 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1.raw.csv 2>&1
  rm -f gpurun_out/$1.ncu-rep
}
cap cheb3d k_chebILi3ENS_6FineOp 2 4
cap residual3d k_residualILi3ENS_6FineOp 1 4
cap cheb3d_stencil k_chebILi3ENS_9StencilOp 1 4
cap cgpq3d k_cg_pqILi3ENS_6FineOp 1 4
cap dgemm k_dgemm_tile 40 1 gmg
unset TMG_PCG_EAGER
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k "regex:k_sens" -s 1 -c 1 -o gpurun_out/full_sens_$R -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 \
  > gpurun_out/full_sens.log 2>&1
digest full_sens_$R
echo done
