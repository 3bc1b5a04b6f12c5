# Round-2 final refresh: GPU tests, smoke, every bench workload, reference arm, launch list and full ncu capture of the headline.
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi > $O/host.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
for wl in "cfg1" "cfg1 --precision bf16" "cfg2" "cfg2 --precision bf16" "cfg5 --steps 3 --warmup 3" "cfg5 --precision fp32 --steps 3 --warmup 3 --e2e-steps 2" "cfg3 --steps 3 --warmup 3"; do
  n=$(echo $wl | tr ' ' '_' | tr -d '-')
  timeout 1200 python bench.py --workload $wl > $O/bench_$n.json 2> $O/bench_$n.err; echo "$wl rc=$?"
done
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "default rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$?"
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-projection --no-comparison > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"umma2_gemm|chain_persistent" -c 3 \
  -o $O/cfg4_full -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-projection --no-comparison > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"chain_persistent" -c 1 \
  -o $O/cfg2_chain_full -f python bench.py --workload cfg2 --precision bf16 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-comparison > $O/ncu_full_cfg2.log 2>&1; echo "ncu cfg2 rc=$?"
timeout 120 python tools/kernel_times.py 262144x2048 bf16 unso 8 bf16 > $O/insitu_cfg4.txt 2>&1
timeout 120 python tools/kernel_times.py 16x2048x512 bf16 unso 8 bf16 > $O/insitu_cfg2_gaussian.txt 2>&1
ls -la $O
