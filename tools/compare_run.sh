#!/bin/bash
# usage: tools/compare_run.sh ROWS COLS
R=$1; C=$2
python tools/compare_engines.py $R $C bf16 /tmp/y_pair.pt
UNSO_ENGINE=1cta python tools/compare_engines.py $R $C bf16 /tmp/y_1cta.pt
python tools/compare_engines.py $R $C fp32 /tmp/y_f64.pt
python - <<'PY'
import torch
a=torch.load('/tmp/y_pair.pt').double(); b=torch.load('/tmp/y_1cta.pt').double(); c=torch.load('/tmp/y_f64.pt').double()
r=lambda u,v: float((u-v).norm()/v.norm())
print("pair vs f64", r(a,c), " 1cta vs f64", r(b,c), " pair vs 1cta", r(a,b))
d=(a-c).abs(); print("max abs err pair", float(d.max()), "argmax row/col", divmod(int(d.argmax()), a.shape[1]))
rowerr=((a-c).norm(dim=1)/c.norm(dim=1)); print("worst rows", rowerr.topk(5))
colerr=((a-c).norm(dim=0)/c.norm(dim=0)); print("worst cols", colerr.topk(5))
PY
