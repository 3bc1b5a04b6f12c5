mkdir -p gpurun_out
{
python tools/kernel_times.py 16x2048x512 fp32 unso
python tools/kernel_times.py 16x2048x512 bf16 unso
python tools/kernel_times.py 16x2048x512 fp32 muon
python tools/kernel_times.py 2048x512 fp32 unso
} > gpurun_out/ktimes.txt 2>&1
tail -5 gpurun_out/ktimes.txt
