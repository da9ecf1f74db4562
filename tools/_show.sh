tail -2 gpurun_out/pytest.log
for c in "$@"; do python3 -c "
import json; d=json.loads(open('gpurun_out/bench_c$c.log').read().strip().splitlines()[-1]); print('c$c', round(d['value'],3), 'GDOF/s', round(d['ms_per_step'],3),'ms', {k:(round(v['ms'],3), round(v['frac_hbm'],3)) for k,v in d['breakdown'].items()})" || tail -3 gpurun_out/bench_c$c.log; done
