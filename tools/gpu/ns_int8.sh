mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32_int8.py tests/test_gpu_guard_bands.py tests/test_gpu_poisoned_workspace.py tests/test_gpu_edge_cases.py -x -q -s > gpurun_out/ns_int8_tests.log 2>&1; tail -3 gpurun_out/ns_int8_tests.log
timeout 300 python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg2_ns.json 2> gpurun_out/bench_cfg2_ns.err; tail -2 gpurun_out/bench_cfg2_ns.err
python -c "import json;d=json.loads(open('gpurun_out/bench_cfg2_ns.json').read().splitlines()[-1]);print(d['ms_per_step'],d.get('ns_comparison'))"
