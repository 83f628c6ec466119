#!/bin/bash
# quick A/B timing on the GPU box: headline + C4 + C3 without e2e extras
python bench.py --steps 10 --warmup 3 --no-extra --cpu-budget 1 > gpurun_out/q_c5.log 2>&1
python bench.py --workload c4 --steps 6 --warmup 2 --no-extra --cpu-budget 1 > gpurun_out/q_c4.log 2>&1
python bench.py --workload c3 --steps 20 --warmup 3 --no-extra --cpu-budget 1 > gpurun_out/q_c3.log 2>&1
for f in gpurun_out/q_c5.log gpurun_out/q_c4.log gpurun_out/q_c3.log; do
python - "$f" <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith('{'):
        d = json.loads(ln); k = d['roofline']['kernels']
        print(sys.argv[1], 'ms/step %.4f' % d['ms_per_step'], 'fwd_core %.4f inv_core %.4f fwd_stages %.4f' % (k['forward_core']['ms'], k['inverse_core']['ms'], k['forward_fft_stages']['ms']))
PY
done
