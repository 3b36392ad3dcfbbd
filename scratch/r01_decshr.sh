for o in "" "--opt shrink_kb_chunk=10" "--opt shrink_kb_chunk=40"; do timeout 300 python bench.py --workload 13b-decode --skip-cpu --skip-e2e --steps 20 --warmup 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$o]', round(d['value']), round(d['ms_per_step'],3), 'shrink', round(r['shrink_ms_per_step'],3))"; done
