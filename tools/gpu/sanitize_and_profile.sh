# One gpurun call: GPU test suite, compute-sanitizer over every route, ncu full capture of the cfg4 kernels.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/host.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = initcheck ] && extra="--track-unused-memory no"
  timeout 1200 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 python tools/sanitize_routes.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/sanitize_summary.txt
  tail -4 gpurun_out/sanitize_$tool.log
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; tail -2 gpurun_out/bench_cfg4.err
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"umma2_gemm|chain_persistent" -c 3 \
  -o gpurun_out/r2_cfg4_full -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-projection > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_full.log
