mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_poisoned_workspace.py -x -q > gpurun_out/chain_tests.log 2>&1; tail -2 gpurun_out/chain_tests.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_q.json 2> gpurun_out/bench_cfg4_q.err; tail -1 gpurun_out/bench_cfg4_q.err
python -c "import json;d=json.loads(open('gpurun_out/bench_cfg4_q.json').read().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'],{k:v['critical_path_ms'] for k,v in d['shard_projection'].items()})"
timeout 300 python bench.py --workload cfg2 --precision bf16 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2bf_q.json 2> gpurun_out/bench_cfg2bf_q.err
python -c "import json;d=json.loads(open('gpurun_out/bench_cfg2bf_q.json').read().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'])"
