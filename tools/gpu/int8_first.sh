mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fp32_int8.py -x -q -s > gpurun_out/int8_tests.log 2>&1; tail -25 gpurun_out/int8_tests.log
timeout 300 python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg2_int8.json 2> gpurun_out/bench_cfg2_int8.err; tail -2 gpurun_out/bench_cfg2_int8.err
python -c "import json;d=json.loads(open('gpurun_out/bench_cfg2_int8.json').read().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'],d['e2e']['ms_per_step'])"
timeout 600 python bench.py --workload cfg5 --precision fp32 --steps 2 --warmup 1 --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_cfg5_fp32_int8.json 2> gpurun_out/bench_cfg5_fp32_int8.err; tail -2 gpurun_out/bench_cfg5_fp32_int8.err
python -c "import json;d=json.loads(open('gpurun_out/bench_cfg5_fp32_int8.json').read().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'],d['ortho_error'],d['ortho_error_reference'])"
