for c in 10 20 40 80 1000; do
timeout 600 python bench.py --workload 13b-decode --skip-cpu --skip-e2e --steps 20 --warmup 5 --opt shrink_kb_chunk=$c 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('chunk $c decode', round(d['value']), round(d['ms_per_step'],3), 'shrink', round(r['shrink_ms_per_step'],3))"
timeout 600 python bench.py --skip-e2e --skip-cpu --steps 3 --opt shrink_kb_chunk=$c 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; g=d['adapter_grads']; print('chunk $c 13b', round(d['value']), round(d['ms_per_step'],1), 'shrink', round(r['shrink_ms_per_step'],2), 'grads', round(g['ms_per_step'],1))"
done
