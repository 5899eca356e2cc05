#!/bin/bash
# quick TF32-kernel iteration on the GPU box: parity tests + C4 / C5 bench lines
python -m pytest -q -p no:cacheprovider -x tests/test_parity_gpu.py -k "tf32" 2>&1 | tail -3
for w in c4 c5; do
  python bench.py --no-cpu --workload $w --steps 50 --tf32 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'], d['dtype'], '%.4g'%d['value'], round(d['ms_per_step'],4), 'K1', round(r['k1_ms_per_launch'],4))"
done
