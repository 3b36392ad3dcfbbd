for o in "" "--opt shrink_mode=2" "--opt shrink_mode=2 --opt shrink_kb_chunk=10" "" "--opt shrink_mode=2"; do
timeout 300 python bench.py --skip-cpu --skip-e2e --steps 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$o]', round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), 'shrink', round(r['shrink_ms_per_step'],2), 'gather', round(r['gather_ms_per_step'],2), d['clocks']['sm_mhz'])"
done
