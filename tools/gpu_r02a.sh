#!/bin/bash
# Round-2 GPU round trip: parity suite, smoke, default bench, config-4 tables.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.log
( time timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 ) 2>&1 | tail -45 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
( time timeout 900 python bench.py ) > gpurun_out/bench.log 2>&1
timeout 600 python tools/iter_breakdown.py --config 4 > gpurun_out/iter_breakdown_c4.txt 2>&1
timeout 600 python tools/roofline_table.py --config 4 > gpurun_out/roofline_c4.txt 2>&1
timeout 600 python tools/iter_breakdown.py --config 3 > gpurun_out/iter_breakdown_c3.txt 2>&1
echo done
