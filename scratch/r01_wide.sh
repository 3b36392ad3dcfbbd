timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python scratch/raster_sweep.py --shapes FFUP_dec --configs "wide_decode=1;wide_decode=0" --iters 20 --warm 5 2>&1 | tail -2
for o in "--opt wide_decode=0" "" "--opt wide_decode=0" ""; do timeout 200 python bench.py --workload 13b-decode --skip-cpu --skip-e2e --steps 20 --warmup 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('decode [$o]', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']))"; done
