timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/m_13b.log 2>&1
timeout 600 python bench.py --workload 7b --skip-cpu > gpurun_out/m_7b.log 2>&1
timeout 600 python bench.py --workload 13b-decode --skip-cpu --steps 20 --warmup 5 > gpurun_out/m_dec.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/m_ref.log 2>&1
for f in m_13b m_7b m_dec m_ref; do tail -1 gpurun_out/$f.log | cut -c1-120; done
