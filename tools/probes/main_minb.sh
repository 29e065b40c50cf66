# main pass resident blocks per SM with 32-sample blocks: FV_MAIN_MINB 6 (default) vs 8 vs 10 (rebuilds on the box)
for m in 6 8 10; do
  make -s -C paper_2209_09965_b200/csrc clean; make -s -j16 -C paper_2209_09965_b200/csrc EXTRA=-DFV_MAIN_MINB=$m > /dev/null 2>&1
  for i in 1 2; do echo "== MINB=$m"; FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/mm_spans.log > /dev/null; python tools/probes/launch_times.py gpurun_out/mm_spans.log 16 | sed -n 3,5p | awk '{printf "%s ", $3} END {print ""}'; done
done
