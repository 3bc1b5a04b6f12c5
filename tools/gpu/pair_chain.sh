mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_poisoned_workspace.py tests/test_gpu_guard_bands.py -x -q > gpurun_out/pair_tests.log 2>&1; tail -2 gpurun_out/pair_tests.log
for i in 1 2; do for v in 0 1; do
UNSO_LIB=exp/dev.so UNSO_CHAIN_PAIR=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-projection > gpurun_out/ab.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().splitlines()[-1]);print('pair=$v',round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['stages_ms'].items()},d['clocks']['sm_mhz'],d['apply_decision'])"
done; done
