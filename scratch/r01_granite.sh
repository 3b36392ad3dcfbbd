for n in 8 16 32 64; do
  timeout 900 python bench.py --workload granite20b --clients $n --steps 2 --warmup 3 --skip-e2e --skip-cpu > gpurun_out/granite_$n.log 2>&1
  tail -1 gpurun_out/granite_$n.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print($n, round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), round(r['frac'],3), 'share', round(r['gemm_share_of_step'],3), d['clocks']['sm_mhz'], d['adapter_grads']['ms_per_step'] if d.get('adapter_grads') else None)"
done
