#!/bin/bash
# chain-stage A/B of exp/base.so vs exp/new.so (default recipe, bf16x3, no truncation) on cfg4, cfg1b, cfg2b
get() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['chain_ms'], d['total_ms'])"; }
for c in cfg4 cfg1b cfg2b; do
  for i in 1 2; do
    echo -n "$c base ";        UNSO_LIB=$(realpath exp/base.so) timeout 200 python tools/stage_profile.py $c 10 | get
    echo -n "$c new ";         UNSO_LIB=$(realpath exp/new.so) timeout 200 python tools/stage_profile.py $c 10 | get
    echo -n "$c new-notrunc "; UNSO_TRUNCATE=0 UNSO_LIB=$(realpath exp/new.so) timeout 200 python tools/stage_profile.py $c 10 | get
  done
done
