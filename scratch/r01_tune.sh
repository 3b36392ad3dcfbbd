for o in "" "--opt gemm_2cta=1" "--opt gemm_2cta=1 --opt group_m=8" "--opt group_m=8" "--opt gemm_2cta=1 --opt pair_n=512"; do
  echo "== $o"
  timeout 600 python bench.py --skip-e2e --skip-cpu --steps 3 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), 'share', round(r['gemm_share_of_step'],3), d['clocks']['sm_mhz'])"
done
