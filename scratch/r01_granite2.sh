for n in 8 16 32 64; do
timeout 900 python bench.py --workload granite20b --clients $n --steps 2 --warmup 3 --skip-e2e --skip-cpu 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; g=d['adapter_grads']; c=r['cublas_same_shapes']
print('| $n |', d['config']['rows_per_fwd_dispatch'], '| **%d** | %.1f | %d | %.3f | %.3f | %.1f | %d | %d |' % (d['value'], d['ms_per_step'], r['achieved'], r['gemm_share_of_step'], c['gemm_time_ratio'], g['ms_per_step'], g['achieved_gbs'], d['clocks']['sm_mhz']))"
done
