# round-2 evidence (third pass: 80-column 4-row tiles, two-row upsample, hit-list composite, 32-sample main blocks):
# full GPU suite + headline parity report, default bench line (CPU baseline + sustained), the
# reference arm, every BASELINE config, C4, smoke, the bench launch list, ncu captures
set -x
mkdir -p gpurun_out
FV_PARITY_REPORT=gpurun_out/r02_headline_parity.json timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/ev_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ev_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/ev_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/ev_bench.log 2>&1; echo "rc=$?" >> gpurun_out/ev_bench.log
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev_ref.log 2>&1; echo "rc=$?" >> gpurun_out/ev_ref.log
for c in c1 c2; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ev_cfg_$c.log 2>&1; done
timeout 900 python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ev_cfg_c5.log 2>&1
timeout 900 python bench.py --config c5 --shard --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ev_cfg_c5s.log 2>&1
timeout 1500 python tools/c4_dense_vs_foveated.py 500 gpurun_out/r02_c4_dense_vs_foveated.json > gpurun_out/ev_c4.log 2>&1
timeout 600 python tools/probes/timeline.py > gpurun_out/ev_timeline.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/ev_ncu_launches.log 2>&1
EXTRA=sm__inst_executed_pipe_tensor_subpipe_hmma.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum,sm__cycles_elapsed.avg,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 1200 ncu --set full --metrics $EXTRA --import-source on --clock-control none -k regex:conv3x3_tc --launch-skip 30 --launch-count 15 -o gpurun_out/r02_conv python tools/profile_frame.py c3 4 > gpurun_out/ev_ncu_conv.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"march_wave|ray_setup|first_list|mask_" --launch-skip 14 --launch-count 7 -o gpurun_out/r02_march python tools/profile_frame.py c3 4 > gpurun_out/ev_ncu_march.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"upsample2|kapply|up3" --launch-skip 26 --launch-count 13 -o gpurun_out/r02_netops python tools/profile_frame.py c3 4 > gpurun_out/ev_ncu_netops.log 2>&1
for r in r02_conv r02_march r02_netops; do ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null; done
ls -la gpurun_out
