for tool in racecheck synccheck; do
timeout 1200 compute-sanitizer --tool $tool --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "batched_equals_solo or decode_size" > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error" gpurun_out/san_$tool.log | head -5
done
