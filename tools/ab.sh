#!/bin/bash
# A/B timing of variant builds: tools/ab.sh CONFIG VAR1 VAR2 ... (base = in-tree library)
cfg=$1; shift
for v in base "$@"; do
  for rep in 1 2; do
    if [ "$v" = base ]; then lib=""; else lib="build/var/$v/liblinedg_b200.so"; fi
    LDG_B200_LIB=$lib timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); b=d['breakdown']
print('$v', 'cfg$cfg', 'step %.4f'%d['ms_per_step'], ' '.join('%s %.4f'%(k,v['ms']) for k,v in b.items()))"
  done
done
