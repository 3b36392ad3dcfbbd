timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plans.py -q -x -k "decode or graph or batched" 2>&1 | tail -2
for o in "--opt lora_overlap=0" "" "--opt lora_overlap=0" ""; do timeout 200 python bench.py --workload 13b-decode --skip-cpu --skip-e2e --steps 20 --warmup 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('decode [$o]', round(d['value']), round(d['ms_per_step'],3))"; done
