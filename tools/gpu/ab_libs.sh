# A/B two builds of the library on one box, alternating: bash tools/gpu/ab_libs.sh A.so B.so [bench args]
mkdir -p gpurun_out
A=$1; B=$2; shift 2
for i in 1 2 3; do for L in $A $B; do
UNSO_LIB=$L timeout 300 python bench.py "$@" --no-cpu-baseline --no-e2e --no-projection > gpurun_out/ab.json 2>/dev/null
python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().splitlines()[-1]);print('$L',round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['stages_ms'].items()},d['clocks']['sm_mhz'],d['clocks']['reasons'])"
done; done
