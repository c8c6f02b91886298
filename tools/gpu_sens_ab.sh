#!/bin/bash
# A/B of the 3D sensitivity kernels (TMG_SENS=gather|stream|brick): parity test + the bench's sensitivity entry
mkdir -p gpurun_out
rm -f gpurun_out/sens_ab.txt
for m in brick gather stream; do
  echo "=== TMG_SENS=$m" >> gpurun_out/sens_ab.txt
  TMG_SENS=$m timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "sensitivity or compliance" 2>&1 | tail -2 >> gpurun_out/sens_ab.txt
  TMG_SENS=$m timeout 900 python bench.py --no-cpu-baseline --steps 5 | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][0])
print('sensitivity', json.dumps(d['sensitivity'])[:330]); print('value', d['value'], 'ms_per_step', d['ms_per_step'], 'compliance', d['leg_results'][0]['compliance'])" >> gpurun_out/sens_ab.txt 2>&1
done
echo done
