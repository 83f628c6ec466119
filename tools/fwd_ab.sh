#!/bin/bash
# A/B of the forward core's consumer-warp count (MWSHT_FWD_CW) at C5 / C5 s2 / C3
for cw in 16 8; do
  for wl in c5s0 c5s2 c3; do
    MWSHT_FWD_CW=$cw timeout 120 python bench.py --workload $wl --steps 10 --warmup 3 --no-extra --cpu-budget 1 > /tmp/ab.json 2>/dev/null
    python -c "
import json,sys
d=json.loads(open('/tmp/ab.json').readline()); k=d['roofline']['kernels']
print('cw=$cw', '$wl', 'ms/step %.4f' % d['ms_per_step'], 'fwd_core %.4f inv_core %.4f err %.2e' % (k['forward_core']['ms'], k['inverse_core']['ms'], d['roundtrip_max_abs_err']))" 2>/dev/null || echo "cw=$cw $wl FAILED/TIMEOUT"
  done
done
