for o in "" "--inplace" "" "--inplace"; do
timeout 600 python bench.py --skip-cpu --skip-e2e --steps 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$o', round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), round(r['frac'],3), 'share', round(r['gemm_share_of_step'],3), 'shrink', round(r['shrink_ms_per_step'],2), 'gather', round(r['gather_ms_per_step'],2), d['clocks'])"
done
