timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/san_smoke.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "batched or decode_size or in_place_device or peer_gpu_routing or rejected" > gpurun_out/san_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/san_tests.log
