#!/bin/bash
# A/B of env switches on the per-config sweep: tools/ab_configs.sh "config2 config3" "DECMG_VTAIL_CTAS=1" "DECMG_VTAIL_CTAS=2" ...
cfgs="$1"; shift
for v in "$@"; do
  env $v python tools/configs_sweep.py $cfgs 2>/tmp/abc.err | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$v', d['config'], 'ms/cycle', d['ms_per_cycle'], 'frac', d['cycle_hbm_frac'], 'cycles', d['cycles_to_1e-8'], 't1e-8', d['time_to_1e-8_s'])
" || tail -3 /tmp/abc.err
done
