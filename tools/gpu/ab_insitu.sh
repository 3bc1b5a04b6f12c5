# A/B of library builds by in-situ (CUPTI) chain kernel time: bash tools/gpu/ab_insitu.sh lib1.so lib2.so ...
for rep in 1 2; do
for lib in "$@"; do
  echo "== $lib (rep $rep)"
  UNSO_LIB=$lib timeout 120 python tools/kernel_times.py 262144x2048 bf16 unso 8 bf16 2>&1 | grep -i "chain_persistent" | head -1
  UNSO_LIB=$lib timeout 120 python tools/kernel_times.py 16x2048x512 bf16 unso 8 bf16 2>&1 | grep -i "chain_persistent" | head -1
done
done
