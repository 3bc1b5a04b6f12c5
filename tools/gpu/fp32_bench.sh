mkdir -p gpurun_out
timeout 600 python bench.py --workload cfg2 --steps 20 --warmup 5 > gpurun_out/bench_cfg2_fp32.json 2> gpurun_out/bench_cfg2_fp32.err; tail -1 gpurun_out/bench_cfg2_fp32.err
timeout 900 python bench.py --workload cfg5 --precision fp32 --steps 3 --warmup 2 --e2e-steps 2 > gpurun_out/bench_cfg5_fp32.json 2> gpurun_out/bench_cfg5_fp32.err; tail -1 gpurun_out/bench_cfg5_fp32.err
timeout 300 python bench.py --workload cfg1 --steps 100 --warmup 5 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; tail -1 gpurun_out/bench_cfg1.err
for f in cfg2_fp32 cfg5_fp32 cfg1; do python -c "import json;d=json.loads(open('gpurun_out/bench_$f.json').read().splitlines()[-1]);print('$f',d['ms_per_step'],d['value'],d['stages_ms'],d['roofline'],d['executed'],d['e2e']['ms_per_step'] if d['e2e'] else None)"; done
