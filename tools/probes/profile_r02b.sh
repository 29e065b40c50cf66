# ncu --set full of one frame's convs (fused K stage) and network elementwise kernels
mkdir -p gpurun_out
EXTRA=sm__inst_executed_pipe_tensor_subpipe_hmma.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum,sm__cycles_elapsed.avg,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 1200 ncu --set full --metrics $EXTRA --import-source on --clock-control none -k regex:conv3x3_tc --launch-skip 30 --launch-count 15 -o gpurun_out/r02b_conv python tools/profile_frame.py c3 4 > gpurun_out/ncu_conv_b.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"upsample2|kapply|up3" --launch-skip 26 --launch-count 13 -o gpurun_out/r02b_netops python tools/profile_frame.py c3 4 > gpurun_out/ncu_netops_b.log 2>&1
for r in r02b_conv r02b_netops; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
done
ls -la gpurun_out | tail -5
