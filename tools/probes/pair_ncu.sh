mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_2cta.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg
for v in 0 1; do
FV_CONV_PAIR=$v timeout 600 ncu --metrics $M --clock-control none -k regex:"conv3x3" --launch-skip 36 --launch-count 18 --csv python tools/profile_frame.py c3 3 > gpurun_out/pair_ncu_$v.csv 2> gpurun_out/pair_ncu_$v.err
done
