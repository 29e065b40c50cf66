# Round-2 profiles: bench launch list (cold, serialised) + ncu --set full of one frame's convs and
# marcher passes (+ tcgen05 operand / tensor-pipe counters), exported as CSV for profiles/
set -x
mkdir -p gpurun_out
EXTRA=sm__inst_executed_pipe_tensor_subpipe_hmma.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
timeout 1200 ncu --set full --metrics $EXTRA --import-source on --clock-control none -k regex:conv3x3_tc --launch-skip 36 --launch-count 18 -o gpurun_out/r02_conv python tools/profile_frame.py c3 4 > gpurun_out/ncu_conv.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"march_wave|ray_setup|first_list|mask_compact" --launch-skip 12 --launch-count 6 -o gpurun_out/r02_march python tools/profile_frame.py c3 4 > gpurun_out/ncu_march.log 2>&1
for r in r02_conv r02_march; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
done
ls -la gpurun_out
