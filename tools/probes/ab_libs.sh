# per-kernel-class times for several library builds: bash tools/probes/ab_libs.sh FIRST COUNT LIB... ("-" = in-tree)
first=$1; count=$2; shift 2
for lib in "$@"; do
  echo "== $lib"
  if [ "$lib" = "-" ]; then timeout 120 python tools/probes/kernel_times.py $first $count | tail -7
  else FV_LIBFOVNET=$lib timeout 120 python tools/probes/kernel_times.py $first $count | tail -7; fi
done
