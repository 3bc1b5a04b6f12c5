mkdir -p gpurun_out
for r in persistent glue; do
UNSO_LIB=exp/dev.so UNSO_BF16_ROUTE=$r timeout 300 python bench.py --workload cfg2 --precision bf16 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_cfg2_$r.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab_cfg2_$r.json').read().splitlines()[-1]);print('$r',d['ms_per_step'],d['stages_ms'],d['ortho_error'][:2],d['ortho_error_reference'][:2])"
done
