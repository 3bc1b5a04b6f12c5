for i in 1 2; do
 echo -n "base "; UNSO_LIB=$(realpath exp/base.so) timeout 200 python tools/stage_profile.py cfg4 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['chain_ms'], d['total_ms'])"
 echo -n "new-f8 "; UNSO_LIB=$(realpath exp/new.so) timeout 200 python tools/stage_profile.py cfg4 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['chain_ms'], d['total_ms'])"
 echo -n "new-bf16x3 "; UNSO_CHAIN=bf16x3 UNSO_LIB=$(realpath exp/new.so) timeout 200 python tools/stage_profile.py cfg4 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['chain_ms'], d['total_ms'])"
done
for c in cfg1b cfg2b; do
 echo -n "$c base "; UNSO_LIB=$(realpath exp/base.so) timeout 200 python tools/stage_profile.py $c 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['chain_ms'], d['total_ms'])"
 echo -n "$c new-f8 "; UNSO_LIB=$(realpath exp/new.so) timeout 200 python tools/stage_profile.py $c 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['chain_ms'], d['total_ms'])"
 echo -n "$c new-bf16x3 "; UNSO_CHAIN=bf16x3 UNSO_LIB=$(realpath exp/new.so) timeout 200 python tools/stage_profile.py $c 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['chain_ms'], d['total_ms'])"
done
