timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for o in "--opt side_shrink=0" "" "--opt side_shrink=0" ""; do timeout 300 python bench.py --workload 13b-decode --skip-cpu --skip-e2e --steps 20 --warmup 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('decode [$o]', round(d['value']), round(d['ms_per_step'],3))"; done
for o in "--opt side_shrink=0" ""; do timeout 300 python bench.py --skip-cpu --skip-e2e --steps 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('13b [$o]', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
