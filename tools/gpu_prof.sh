timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
python tools/profile_case.py --config 1 --iters 200 > gpurun_out/plain.log 2>&1; cat gpurun_out/plain.log
TMG_PCG_EAGER=1 python tools/profile_case.py --config 1 --iters 20 --reps 1 > gpurun_out/plain2.log 2>&1 && TMG_PCG_EAGER=1 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 3000 --csv --log-file gpurun_out/launches_warm.csv python tools/profile_case.py --config 1 --iters 20 --reps 1 > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log
