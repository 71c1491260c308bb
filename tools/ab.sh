#!/bin/bash
# A/B timing of env switches on the headline bench (no CPU baseline, no scale line):
#   tools/ab.sh "DECMG_FUSE_PC=0" "DECMG_FUSE_PC=1" ...
for v in "$@"; do
  for rep in 1 2; do
    env $v python bench.py --no-cpu-baseline --no-scale-config --steps 20 > /tmp/ab.json 2>/tmp/ab.err || { echo "$v FAILED"; tail -3 /tmp/ab.err; continue; }
    python - "$v" <<'PY'
import json, sys
d = json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1])
r = d['roofline']
print(sys.argv[1], f"ms/step {d['ms_per_step']:.4f}", f"value {d['value']/1e9:.2f} G", f"cycle frac {d['cycle_roofline']['frac_measured_peak']:.3f}",
      {k: round(v / d['steps'], 3) for k, v in r['classes_ms'].items()}, f"e2e {d['e2e']['value']/1e9:.2f} G")
PY
  done
done
