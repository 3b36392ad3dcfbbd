timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"seg_gemm|gather_rows|lora_shrink|copy_rows" -s 1500 -c 1300 --csv --log-file /tmp/dl.csv python bench.py --workload 13b-decode --steps 1 --warmup 3 --skip-e2e --skip-cpu --graph 0 > /tmp/dl.log 2>&1
echo rc=$?
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(l for l in open('/tmp/dl.csv') if not l.startswith('==')))
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows:
    if r.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    n = r['Kernel Name'].split('(')[0].split('<')[0].replace('void ', '').strip()
    if 'seg_gemm' in r['Kernel Name']:
        n = r['Kernel Name'].split('(')[0].replace('void ', '').strip()
    v = float(r['Metric Value'].replace(',', ''))
    unit = r['Metric Unit']
    v = v / 1e3 if unit == 'nsecond' else v if unit == 'usecond' else v * 1e3
    tot[n] += v; cnt[n] += 1
all_ = sum(tot.values())
with open('gpurun_out/dec_launches.md', 'w') as f:
    f.write('| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|\n')
    for n, v in sorted(tot.items(), key=lambda x: -x[1]):
        f.write(f'| {n} | {cnt[n]} | {v:.0f} | {v / cnt[n]:.1f} | {v / all_:.3f} |\n')
print(open('gpurun_out/dec_launches.md').read())
PY
