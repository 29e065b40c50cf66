mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"march_wave_shadow_dir|march_wave_main_list|march_wave_composite" --launch-skip 6 --launch-count 3 -o gpurun_out/r02c_march python tools/profile_frame.py c3 4 > gpurun_out/ncu_march_c.log 2>&1
ncu -i gpurun_out/r02c_march.ncu-rep --page raw --csv > gpurun_out/r02c_march.raw.csv 2>/dev/null
ncu -i gpurun_out/r02c_march.ncu-rep --page source --csv -k regex:march_wave_shadow_dir > gpurun_out/r02c_shadow_source.csv 2>/dev/null
ncu -i gpurun_out/r02c_march.ncu-rep --page source --csv -k regex:march_wave_main_list > gpurun_out/r02c_main_source.csv 2>/dev/null
ncu -i gpurun_out/r02c_march.ncu-rep --page details --csv > gpurun_out/r02c_march_details.csv 2>/dev/null
