mkdir -p gpurun_out
for v in _a _b _c; do
  for c in 3 4; do
    TMG_LIB=$PWD/paper_2001_01655_b200/lib/libtopomg_b200$v.so timeout 600 python tools/roofline_table.py --config $c --reps 20 2>&1 | grep matrix_free | head -2 > gpurun_out/tile$c$v.txt
    TMG_LIB=$PWD/paper_2001_01655_b200/lib/libtopomg_b200$v.so timeout 300 python tools/iter_breakdown.py --config $c --iters 100 2>&1 | grep PCG >> gpurun_out/tile$c$v.txt
  done
done
