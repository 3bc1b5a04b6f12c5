#!/bin/bash
# fp32-mode (fp64 engine) stage A/B: tools/ab_fp32.sh libA libB ...
get() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gram', d['gram_ms'], 'chain', d['chain_ms'], 'apply', d['apply_ms'], 'total', round(d['total_ms'],3))"; }
for c in "cfg1f 10" "cfg2f 3" "cfg5f 1 1"; do
  for L in "$@"; do echo -n "$c $L "; UNSO_LIB=$(realpath exp/$L.so) timeout 300 python tools/stage_profile.py $c | get; done
done
