mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_guard_bands.py tests/test_gpu_parity.py::test_cfg4_full_size_rows_against_oracle -q -s > gpurun_out/guard_tests.log 2>&1; tail -3 gpurun_out/guard_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -4 gpurun_out/smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 --cpu-full > gpurun_out/bench_cfg4_cpufull.json 2> gpurun_out/bench_cfg4_cpufull.err; tail -2 gpurun_out/bench_cfg4_cpufull.err
cp profiles/cpu_full_workload.json gpurun_out/ 2>/dev/null; ls profiles/cpu_full_workload.json
