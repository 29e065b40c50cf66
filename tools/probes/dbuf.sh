mkdir -p gpurun_out
rm -f gpurun_out/dbuf_ab.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/dbuf_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/dbuf_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/dbuf_ab.log; }
run s1 ""
run f1 "FV_KCHAIN_SPLIT=2 FV_KCHAIN_AT=1"
run f12 "FV_KCHAIN_SPLIT=2 FV_KCHAIN_AT=12"
run f13 "FV_KCHAIN_SPLIT=2 FV_KCHAIN_AT=13"
run f9 "FV_KCHAIN_SPLIT=2 FV_KCHAIN_AT=9"
run s1b ""
run f12b "FV_KCHAIN_SPLIT=2 FV_KCHAIN_AT=12"
