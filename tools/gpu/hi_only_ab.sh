mkdir -p gpurun_out
for v in 0 2 3 4; do
UNSO_LIB=exp/dev.so UNSO_PCHAIN_HI_ONLY=$v python tools/hi_only_probe.py 2>/dev/null
for wl in "cfg4" "cfg2 --precision bf16"; do
UNSO_LIB=exp/dev.so UNSO_PCHAIN_HI_ONLY=$v timeout 300 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-projection > gpurun_out/ab.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().splitlines()[-1]);print('  $wl hi_only=$v',round(d['ms_per_step'],4),'chain',round(d['stages_ms']['chain'],4),d['clocks']['sm_mhz'])"
done; done
