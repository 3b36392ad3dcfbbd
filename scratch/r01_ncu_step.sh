# ncu --set full over one block's forward GEMMs, the LM head fwd/bwd and one block's backward GEMMs
# of the 13B bench step (eager plans), plus the adapter-gradient kernels.
B="python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu --graph 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm -s 1446 -c 6 -o gpurun_out/step_fwd $B > gpurun_out/ncu_step_fwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm -s 1686 -c 8 -o gpurun_out/step_head_bwd $B > gpurun_out/ncu_step_bwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lora_grad|ia3_grad|lora_shrink" -s 6 -c 3 -o gpurun_out/grads_full2 python scratch/grads_bench.py > gpurun_out/ncu_grads2.log 2>&1
tail -2 gpurun_out/ncu_step_fwd.log gpurun_out/ncu_step_bwd.log gpurun_out/ncu_grads2.log
