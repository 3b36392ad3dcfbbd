for v in "" scratch/variants/st5.so scratch/variants/st3.so ""; do
  echo "== lib $v" >> gpurun_out/st_time.log
  SS_B200_LIB=$v python scratch/raster_sweep.py --shapes Q_dec,FFDOWN_dec,HEAD_dec --iters 20 --warm 5 --configs "pf_depth=0" >> gpurun_out/st_time.log 2>&1
done
cat gpurun_out/st_time.log
