# round-end measurement set: tests, smoke, default bench, all configs, ncu launch list + captures
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t_gpu.log 2>&1; tail -1 gpurun_out/t_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log > gpurun_out/bench_line.json
rm -f gpurun_out/cfg_results.txt; bash tools/probes/configs.sh
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r01_bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"march_wave|ray_setup|first_list" --launch-skip 10 --launch-count 5 -o gpurun_out/prof_march_r01f python tools/profile_frame.py c3 3 > gpurun_out/ncu_m.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:conv3x3_tc --launch-skip 18 --launch-count 18 -o gpurun_out/prof_conv_r01f python tools/profile_frame.py c3 3 > gpurun_out/ncu_c.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"kapply|up3|upsample2|mask_compact" --launch-skip 14 --launch-count 14 -o gpurun_out/prof_netops_r01f python tools/profile_frame.py c3 3 > gpurun_out/ncu_n.log 2>&1
