#!/bin/bash
# Round-end check: full parity suite, smoke, both bench arms, the coarse GEMV capture.
mkdir -p gpurun_out
R=r02
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s ) 2>&1 | grep -E "k=|passed|failed|Error|real" > gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
( time timeout 900 python bench.py --steps 20 --warmup 5 ) > gpurun_out/bench_$R.log 2>&1
( time timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/bench_ref_$R.log 2>&1
export TMG_PCG_EAGER=1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:k_gemv_split" -s 2 -c 1 -o gpurun_out/full_gemv_$R -f \
    python tools/profile_case.py --config 1 --iters 3 --reps 1 --legs gmg > gpurun_out/full_gemv.log 2>&1
ncu -i gpurun_out/full_gemv_$R.ncu-rep --page details > gpurun_out/full_gemv_$R.details.txt 2>&1
ncu -i gpurun_out/full_gemv_$R.ncu-rep --page raw --csv > gpurun_out/full_gemv_$R.raw.csv 2>&1
rm -f gpurun_out/full_gemv_$R.ncu-rep
echo done
