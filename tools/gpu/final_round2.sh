# Round-2 refresh: GPU tests, smoke, every bench workload (headline default last), launch list of the headline.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1; tail -1 gpurun_out/pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for wl in "cfg1" "cfg1 --precision bf16" "cfg2" "cfg2 --precision bf16" "cfg5 --steps 3 --warmup 3" "cfg5 --precision fp32 --steps 3 --warmup 3 --e2e-steps 2" "cfg3 --steps 3 --warmup 3"; do
  n=$(echo $wl | tr ' ' '_' | tr -d '-')
  timeout 1200 python bench.py --workload $wl > gpurun_out/bench_$n.json 2> gpurun_out/bench_$n.err; echo "$wl rc=$?"
done
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference rc=$?"
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-projection --no-comparison > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
