# C1 (64^3, 256^2): the round's new defaults one at a time reverted
run() { env "$@" python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline --no-sustained 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['value'],1), round(d['e2e']['value'],1))"; }
for i in 1 2; do
run X=0; run FV_N80_R=2; run FV_MAIN_U=2; run FV_COMP_HITS=0; run FV_UP_ROWS=1; run FV_N80_R=2 FV_MAIN_U=2 FV_COMP_HITS=0 FV_UP_ROWS=1
done
bash tools/probes/mask_inc.sh
