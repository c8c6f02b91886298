#!/bin/bash
# full parity suite (checkpoints printed), coarse-inverse timings (Cholesky vs Gauss-Jordan), ncu of the big tile GEMM
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s ) 2>&1 | grep -E "k=|passed|failed|Error|real" > gpurun_out/pytest_gpu_all.log
rm -f gpurun_out/setup_r02.txt
for m in chol gj; do
  echo "=== TMG_COARSE=$m" >> gpurun_out/setup_r02.txt
  TMG_COARSE=$m TMG_VERBOSE=1 timeout 600 python tools/profile_case.py --config 1 --iters 5 --legs gmg 2>&1 | grep -E "coarse|setup_ms" >> gpurun_out/setup_r02.txt
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --kernel-name-base function -k regex:"k_dgemm_tile|k_chol|k_sym_from" \
  --log-file gpurun_out/launches_chol_r02.csv python tools/profile_case.py --config 1 --iters 2 --reps 1 --legs gmg > gpurun_out/ncu_chol.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:k_dgemm_tileILb1ELb0" -c 1 -o gpurun_out/full_dgemm_gram_r02 -f \
    python tools/profile_case.py --config 1 --iters 2 --reps 1 --legs gmg > gpurun_out/full_dgemm_gram.log 2>&1
ncu -i gpurun_out/full_dgemm_gram_r02.ncu-rep --page details > gpurun_out/full_dgemm_gram_r02.details.txt 2>&1
ncu -i gpurun_out/full_dgemm_gram_r02.ncu-rep --page raw --csv > gpurun_out/full_dgemm_gram_r02.raw.csv 2>&1
rm -f gpurun_out/full_dgemm_gram_r02.ncu-rep
echo done
