# quick loop for persistent-chain work: parity subsets, cfg2/cfg4 traces (timing build in exp/), quick benches
mkdir -p gpurun_out
T=${1:-iter}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_poisoned_workspace.py tests/test_gpu_edge_cases.py -x -q > gpurun_out/${T}_tests.log 2>&1; tail -2 gpurun_out/${T}_tests.log
if [ -f exp/timing.so ]; then
  UNSO_LIB=exp/timing.so timeout 120 python tools/chain_trace.py 512 2048 16 > gpurun_out/${T}_trace_cfg2.txt 2>&1; head -12 gpurun_out/${T}_trace_cfg2.txt; grep "phase A" gpurun_out/${T}_trace_cfg2.txt | head -1
  UNSO_LIB=exp/timing.so timeout 120 python tools/chain_trace.py > gpurun_out/${T}_trace_cfg4.txt 2>&1; head -12 gpurun_out/${T}_trace_cfg4.txt; grep "phase A" gpurun_out/${T}_trace_cfg4.txt | head -1
fi
timeout 300 python bench.py --workload cfg2 --precision bf16 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_cfg2bf.json 2> gpurun_out/${T}_bench.err
python -c "import json;d=json.loads(open('gpurun_out/${T}_bench_cfg2bf.json').read().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'])"
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_cfg4.json 2>> gpurun_out/${T}_bench.err
python -c "import json;d=json.loads(open('gpurun_out/${T}_bench_cfg4.json').read().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'],d['clocks'])"
timeout 120 python tools/kernel_times.py 262144x2048 bf16 unso 5 bf16 2>&1 | grep -i "chain_persistent" | head -1
timeout 120 python tools/kernel_times.py 16x2048x512 bf16 unso 5 bf16 2>&1 | grep -i "chain_persistent" | head -1
