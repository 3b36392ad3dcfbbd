timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python scratch/raster_sweep.py --shapes Q_dec,FFUP_dec,FFDOWN_dec,HEAD_dec --configs "raster=0" --iters 20 --warm 5 2>&1 | tail -4
for i in 1 2; do timeout 200 python bench.py --workload 13b-decode --skip-cpu --skip-e2e --steps 20 --warmup 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('decode', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']))"; done
