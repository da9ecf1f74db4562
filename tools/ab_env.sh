#!/bin/bash
# A/B timing of environment settings: tools/ab_env.sh CONFIG "ENV=..." "ENV=..." (first = baseline "")
cfg=$1; shift
for e in "" "$@"; do
  for rep in 1 2; do
    env $e timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); b=d['breakdown']
print('[$e]', 'cfg$cfg', 'step %.4f'%d['ms_per_step'], ' '.join('%s %.4f'%(k,v['ms']) for k,v in b.items()))"
  done
done
