for rep in 1 2; do
for o in "" "--opt l2_hints=0" "--opt raster=-1" "--opt pair_n=512" "--opt group_m=8" "--opt group_m=32"; do
timeout 600 python bench.py --skip-cpu --skip-e2e --steps 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$o]', round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), round(r['frac'],3), 'shrink', round(r['shrink_ms_per_step'],2), 'gather', round(r['gather_ms_per_step'],2), d['clocks']['sm_mhz'])"
done; done
