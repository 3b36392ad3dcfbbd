timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for o in "--opt stream_pdl=0" "" "--opt stream_pdl=0" ""; do timeout 200 python bench.py --workload 13b-decode --skip-cpu --skip-e2e --steps 20 --warmup 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('decode [$o]', round(d['value']), round(d['ms_per_step'],3))"; done
