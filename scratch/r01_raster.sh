python scratch/raster_sweep.py > gpurun_out/raster_time.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:seg_gemm --csv --log-file gpurun_out/raster_ncu.csv python scratch/raster_sweep.py --iters 1 --warm 0 > gpurun_out/raster_ncu_run.log 2>&1
for kn in "5120 5120" "5120 13824" "13824 5120" "5120 32000"; do
  python scratch/prof_shape.py $kn 64 0 0 16 10 >> gpurun_out/decode_time.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_gemm -c 1 -o gpurun_out/decode_q python scratch/prof_shape.py 5120 5120 64 0 0 16 1 > gpurun_out/ncu_dec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_gemm -c 1 -o gpurun_out/decode_ffdown python scratch/prof_shape.py 13824 5120 64 0 0 16 1 >> gpurun_out/ncu_dec.log 2>&1
cat gpurun_out/raster_time.log gpurun_out/decode_time.log
