timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/n_13b.log 2>&1; tail -1 gpurun_out/n_13b.log | cut -c1-200
timeout 600 python bench.py --impl reference > gpurun_out/n_ref.log 2>&1; tail -1 gpurun_out/n_ref.log | cut -c1-150
