mkdir -p gpurun_out
make -s -C paper_2209_09965_b200/csrc clean
make -s -C paper_2209_09965_b200/csrc -j16 EXTRA=-DFV_CONV_PROFILE=1 > gpurun_out/build_prof.log 2>&1
FV_CONV_PAIR=1 FV_CONV_PROF=1 FV_GRAPH=0 timeout 600 python tools/profile_frame.py c3 3 > gpurun_out/pair_waits.log 2>&1
