#!/bin/bash
# Round-end style validation: parity suite, smoke, bench (both arms).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -6 > gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/final_bench_ref.log 2>&1
echo done
