for o in "--opt side_shrink=0" "" "--opt side_shrink=0" ""; do timeout 300 python bench.py --workload 13b-decode --skip-cpu --steps 5 --e2e-steps 3 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$o]', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],1))"; done
nproc; cat /proc/cpuinfo | grep "model name" | head -1
