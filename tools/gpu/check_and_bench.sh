mkdir -p gpurun_out
free -g > gpurun_out/host.txt; nproc >> gpurun_out/host.txt; nvidia-smi >> gpurun_out/host.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for wl in cfg4 cfg1 cfg2; do timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; done
timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 2 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --workload cfg5 --precision fp32 --steps 2 --warmup 1 --e2e-steps 2 > gpurun_out/bench_cfg5_fp32.json 2> gpurun_out/bench_cfg5_fp32.err
timeout 900 python bench.py --workload cfg3 --steps 3 --warmup 2 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
tail -2 gpurun_out/*.err
