#!/bin/bash
# A/B of the plain inverse core's consumer-warp count (MWSHT_INV_CW): C2 and an
# L=1024 spin-2 map (c5s2 workload with --band-limit 1024)
for cw in 16 8; do
  for args in "--workload c2" "--workload c5s2 --band-limit 1024" "--workload c5s2 --band-limit 512"; do
    MWSHT_INV_CW=$cw timeout 120 python bench.py $args --steps 20 --warmup 3 --no-extra --cpu-budget 1 > /tmp/ab.json 2>/dev/null
    python -c "
import json
d=json.loads(open('/tmp/ab.json').readline()); k=d['roofline']['kernels']
print('cw=$cw', '$args', 'ms/step %.4f' % d['ms_per_step'], 'fwd_core %.4f inv_core %.4f err %.2e' % (k['forward_core']['ms'], k['inverse_core']['ms'], d['roundtrip_max_abs_err']))" 2>/dev/null || echo "cw=$cw $args FAILED/TIMEOUT"
  done
done
