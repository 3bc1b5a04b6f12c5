"""Dev tool: warm, in-situ per-kernel device times of one orthogonalize call (CUPTI activity records
through torch.profiler, no replay / serialisation -- unlike an ncu launch list).

usage: python tools/kernel_times.py SHAPE PRECISION [method] [calls] [input dtype: fp32|bf16]
       e.g. 16x2048x512 fp32 unso 5   |   2048x512 fp32 muon   |   262144x2048 bf16 unso 5 bf16
Also prints the device timeline of the last call (start offset, duration, gap to the previous activity).
"""
import collections
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2602_02500_b200 as U  # noqa: E402


def main():
    shape = [int(s) for s in sys.argv[1].split("x")]
    prec = sys.argv[2]
    method = sys.argv[3] if len(sys.argv) > 3 else "unso"
    calls = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    if method == "unso":
        spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    elif method == "muon":
        spec = U.MethodSpec(U.MethodKind.MUON_NS, iterations=5)
    else:
        spec = U.MethodSpec(U.MethodKind.ORIGINAL_NS, iterations=6)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(*shape, generator=g, device="cuda")
    if len(sys.argv) > 5 and sys.argv[5] == "bf16":
        x = x.to(torch.bfloat16)
    for _ in range(3):
        U.orthogonalize(x, spec, precision=prec)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(calls):
            U.orthogonalize(x, spec, precision=prec)
        torch.cuda.synchronize()
    agg = collections.OrderedDict()
    first = last = None
    for ev in prof.events():
        if ev.device_type != torch.autograd.DeviceType.CUDA:
            continue
        name = ev.name.split("(")[0][:72]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ev.device_time
        s, e = ev.time_range.start, ev.time_range.end
        first = s if first is None else min(first, s)
        last = e if last is None else max(last, e)
    tot = 0.0
    print(f"{sys.argv[1]} {prec} {method}: per call (mean of {calls})")
    for k, (c, t) in agg.items():
        tot += t
        print(f"  {k:72s} {c / calls:5.1f} x {t / c:8.2f} us = {t / calls:9.2f} us")
    print(f"  kernels {tot / calls:.1f} us per call, span {(last - first) / calls:.1f} us per call")
    evs = sorted((ev for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA),
                 key=lambda ev: ev.time_range.start)
    per = len(evs) // calls
    tail = evs[-per:]
    t0, prev_end = tail[0].time_range.start, None
    print("  timeline of the last call: start(us)  dur(us)  gap(us)  name")
    for ev in tail:
        s, e = ev.time_range.start, ev.time_range.end
        gap = 0.0 if prev_end is None else s - prev_end
        print(f"    {s - t0:9.1f} {e - s:9.1f} {gap:8.1f}  {ev.name.split('(')[0][:60]}")
        prev_end = e


if __name__ == "__main__":
    main()
