for o in "" "--opt shrink_kb_chunk=10" "" "--opt shrink_kb_chunk=10"; do timeout 300 python bench.py --skip-cpu --skip-e2e --steps 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('13b [$o]', round(d['value']), round(d['ms_per_step'],1), 'shrink', round(r['shrink_ms_per_step'],2), d['clocks']['sm_mhz'])"; done
