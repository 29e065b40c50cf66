# A/B two library builds on the per-kernel-class probe: bash tools/probes/ab_lib.sh OLD.so FIRST COUNT [rounds]
old=$1; first=$2; count=$3; rounds=${4:-2}
for i in $(seq $rounds); do
  echo "== old"; FV_LIBFOVNET=$old timeout 120 python tools/probes/kernel_times.py $first $count | tail -7
  echo "== new"; timeout 120 python tools/probes/kernel_times.py $first $count | tail -7
done
