for w in cfg1 mt lm; do for i in 1 2; do
timeout 300 python bench.py --workload $w --no-cpu-baseline --no-clocks > gpurun_out/ab.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$w', d['ms_per_step'], d['e2e']['ms_per_step'], round(d['e2e']['value']/1e6,2))"
done; done
MOE_HOST_PIPE_PROF=1 timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-clocks 2>&1 >/dev/null | grep "host pipe" | tail -4
