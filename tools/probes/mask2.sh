mkdir -p gpurun_out
rm -f gpurun_out/mask2_ab.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "mask or scatter or pipelined or cmax or direct or shard" > gpurun_out/mask2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/mask2_tests.log
timeout 900 python -m pytest tests/test_headline_parity.py -q -m gpu -k "masks" >> gpurun_out/mask2_tests.log 2>&1
echo "headline rc=$?" >> gpurun_out/mask2_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/mask2_ab.log; }
run m2 ""; run m1 "FV_MASK_2PASS=0"; run m2b ""; run m1b "FV_MASK_2PASS=0"
