for o in "" "--opt tile_n=128" "--opt tile_n=256"; do
  echo "== $o"
  timeout 600 python bench.py --workload 13b-decode --skip-cpu --steps 20 --warmup 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],3), 'gemm', round(r['achieved']), r['unit'], round(r['frac'],3), 'share', round(r['gemm_share_of_step'],3), 'shrink', round(r['shrink_ms_per_step'],3), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])"
done
