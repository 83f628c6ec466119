#!/bin/bash
# A/B of the inverse cores' consumer-warp count: paired (MWSHT_PINV_CW) at
# C3 / single spin-0 maps, plain (MWSHT_INV_CW) at spin 2
VAR=${VAR:-MWSHT_PINV_CW}
for cw in 16 8; do
  while read -r args; do
    env $VAR=$cw timeout 120 python bench.py $args --steps 20 --warmup 3 --no-extra --cpu-budget 1 > /tmp/ab.json 2>/dev/null
    python -c "
import json
d=json.loads(open('/tmp/ab.json').readline()); k=d['roofline']['kernels']
print('$VAR=$cw', '$args', 'ms/step %.4f' % d['ms_per_step'], 'fwd_core %.4f inv_core %.4f err %.2e' % (k['forward_core']['ms'], k['inverse_core']['ms'], d['roundtrip_max_abs_err']))" 2>/dev/null || echo "$VAR=$cw $args FAILED/TIMEOUT"
  done <<ARGS
${CASES:---workload c3
--workload c5s0 --band-limit 512
--workload c5s0 --band-limit 1024
--workload c5s0 --band-limit 2048}
ARGS
done
