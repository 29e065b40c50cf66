mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "forward or end_to_end or pipelined" > gpurun_out/ups_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ups_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/ups_ab.log; }
run u2 ""
run u2b ""
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"mask_compact|upsample2" --launch-skip 6 --launch-count 4 -o gpurun_out/r02c_mask python tools/profile_frame.py c3 4 > gpurun_out/ncu_mask.log 2>&1
ncu -i gpurun_out/r02c_mask.ncu-rep --page raw --csv > gpurun_out/r02c_mask.raw.csv 2>/dev/null
ncu -i gpurun_out/r02c_mask.ncu-rep --page source --csv -k regex:mask_compact > gpurun_out/r02c_mask_source.csv 2>/dev/null
