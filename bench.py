#!/usr/bin/env python
"""UNSO orthogonalization benchmark on B200 (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[3], the config its 1/2/4/8-GPU metric and the
north_star's scaling target are quoted on): one tall bf16 matrix 262144 x 2048,
i.i.d. N(0,1) (seeded synthetic), orthogonalized with the shipped order-14 UNSO
polynomial in bf16 mode (tcgen05 bf16 tensor cores; SYRK Gram; bf16x3 C-form chain
with data-dependent truncation; adaptive single-term / bf16x2 apply of the shifted P).  With --gpus N > 1 (torchrun) the rows are sharded along the long side:
local Gram -> one NCCL all-reduce of the 2048 x 2048 Gram -> redundant P(A) ->
local apply (strong scaling: total work fixed).

A step = one full orthogonalization (preprocess + chain + apply) of the matrix.
value   = reference-model FLOPs (kernel_model_flops, ortho.py:313-335) per second, whole job.
e2e     = the same metric through the public API with the input in pinned host memory
          and the result copied back to pinned host memory inside the timed region.
--impl reference times the CPU oracle (numpy fp64 restatement of the reference) on a
bounded row sample of the same workload on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "UNSO orthogonalization TFLOP/s & matrices/s (% bf16 tensor peak), 1/2/4/8 B200"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--rows", type=int, default=262144)
    ap.add_argument("--cols", type=int, default=2048)
    ap.add_argument("--precision", choices=["bf16", "fp32"], default="bf16")
    ap.add_argument("--collective", choices=["nccl", "nvlink"], default="nccl",
                    help="N > 1: Gram all-reduce through NCCL, or the peer-memory reduction (unso_gram_push/...)")
    ap.add_argument("--apply-terms", type=int, choices=[1, 2], default=None,
                    help="bf16 apply split: default adaptive per matrix (device-side bound)")
    ap.add_argument("--e2e-steps", type=int, default=30,
                    help="pipelined e2e steps (fill and drain of the three-stream pipeline amortised over them)")
    ap.add_argument("--cpu-sample-rows", type=int, default=65536,
                    help="rows of the cpu_baseline sample (~10 s of OpenBLAS fp64 on the GPU box host)")
    ap.add_argument("--ref-sample-rows", type=int, default=8192)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run the row-sharded multi-rank path (process group, Gram reduction) even at world size 1; "
                         "used to exercise the N > 1 code under torchrun on a single GPU")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d, "measured"
    return dict(FALLBACK_PEAKS), "fallback"


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, ValueError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                self.samples.append((time.time(), float(parts[0]), float(parts[1]), parts[3:7]))
            except ValueError:
                continue

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=5)

    def summary(self, t0: float, t1: float):
        win = [s for s in self.samples if t0 - 0.05 <= s[0] <= t1 + 0.05] or self.samples
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = sorted({n for s in win for n, v in zip(self.NAMES, s[3]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(s[1] for s in win), "sm_max_mhz": max(s[2] for s in win),
                "reasons": reasons, "samples": len(win)}


def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("internal_api") in ("openblas", "mkl")]
        if n and n[0]:
            return int(n[0])
    except Exception:
        pass
    return os.cpu_count() or 1


def cpu_oracle_sample(rows: int, cols: int, seed: int, bf16: bool = True):
    """Time the CPU oracle (numpy fp64 port of the reference) on a rows x cols sample."""
    import numpy as np
    import torch
    from oracle import unso_oracle as O
    g = torch.Generator().manual_seed(seed)
    m = torch.randn(rows, cols, generator=g)
    if bf16:
        m = m.to(torch.bfloat16)
    m = m.double().numpy()
    t0 = time.perf_counter()
    O.run(m, "unso")
    dt = time.perf_counter() - t0
    h, w = min(rows, cols), max(rows, cols)
    return O.model_flops("unso", h, w), dt


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores, rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    rows = min(args.ref_sample_rows, args.rows)
    cols = args.cols
    f = None
    for _ in range(args.warmup):
        f, _ = cpu_oracle_sample(rows, cols, 7)
    times = []
    for i in range(args.steps):
        f, dt = cpu_oracle_sample(rows, cols, 7 + i)
        times.append(dt)
    total = sum(times)
    value = f * len(times) / total / 1e12
    cores = cpu_threads()
    sample = (f"{rows}x{cols} row sample of the {args.rows}x{cols} workload (bf16-rounded N(0,1), fp64 numpy/OpenBLAS "
              f"oracle restating unso.ortho.orthogonalize), {args.steps} timed steps")
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"configs[3] UNSO {args.rows}x{cols} (CPU sample {rows}x{cols})",
                   "global_batch": 1, "shape": [args.rows, cols], "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2602_02500_b200 as U
    from paper_2602_02500_b200 import _native as N
    from paper_2602_02500_b200.distributed import orthogonalize_row_sharded, row_shard_bounds

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or args.sharded
    if sharded:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if sharded:
            dist.barrier()

    rows, cols = args.rows, args.cols
    h, w = (cols, rows) if rows > cols else (rows, cols)
    r0, r1 = row_shard_bounds(rows, world, rank)
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(r1 - r0, cols, generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16
                                                                                      if args.precision == "bf16"
                                                                                      else torch.float32)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), precision=args.precision,
                        apply_terms=args.apply_terms)
    y = torch.empty_like(x)

    def step():
        if not sharded:
            U.orthogonalize(x, spec, out=y, check=False)
        else:
            orthogonalize_row_sharded(x, spec, out=y, check=False, collective=args.collective)

    # ---- correctness gate (untimed): status + orthogonality of the output
    apply_info = None
    if not sharded:
        res = U.orthogonalize(x, spec, out=y, check=True)
        launches_per_step = res.launches
        apply_info = res.info[0] if res.info else None
    else:
        orthogonalize_row_sharded(x, spec, out=y, check=True, collective=args.collective)
        launches_per_step = None
    torch.cuda.synchronize()
    if not sharded:
        ortho_err = float(U.ortho_error_device(y)[0])
    else:   # untimed check: ||Y^T Y - I||_F with the shard Grams summed over the group
        yf = y.float()
        gy = (yf.T @ yf) if rows > cols else (yf @ yf.T)
        dist.all_reduce(gy)
        gy -= torch.eye(gy.shape[0], device=dev)
        ortho_err = float(torch.linalg.norm(gy))
    # The reference's own orthogonality error on this input: Y_ref = X P(X^T X) has singular values
    # g(sigma(X)) (the scalar map, ortho.py:286-310), so ||Y_ref^T Y_ref - I||_F follows from the
    # spectrum of X (fp64 Gram, summed over the shards, eigenvalues on the device; untimed).
    xg = x.double()
    gx = (xg.T @ xg) if rows > cols else (xg @ xg.T)
    del xg
    if sharded:
        dist.all_reduce(gx)
    sx = torch.sqrt(torch.linalg.eigvalsh(gx).clamp_min(0.0)).cpu().numpy()
    del gx
    sy = U.scalar_map(spec)(sx / float((sx ** 4).sum()) ** 0.25)
    ortho_ref = float(np.sqrt(((sy ** 2 - 1.0) ** 2).sum()))
    if launches_per_step is None:
        # our kernels per step, from the library's per-call counters: the Gram stage (or the
        # push / reduce / wait kernels of the peer-memory reduction) plus the finish stage
        if args.collective == "nccl":
            g = U.distributed.native_gram(x, spec, None)
            launches_per_step = N.launch_count()
        else:
            red = U.distributed._nvlink_reducer(cols, x.shape[0], None, dev)
            red.push(x, spec, None)
            launches_per_step = N.launch_count()
            red.reduce()
            launches_per_step += N.launch_count()
            g = red.wait()
            launches_per_step += N.launch_count()
        U.distributed.native_finish(x, g, spec, None, y)
        launches_per_step += N.launch_count()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    barrier()

    peaks, peaks_src = load_peaks()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    stream = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = N.StageProfiler(args.steps) if not sharded else None
    if prof:
        prof.__enter__()
    barrier()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.time()
    barrier()
    ms_local = ev0.elapsed_time(ev1)
    stage_ms = prof.read() if prof else None
    if prof:
        prof.__exit__(None, None, None)
    time.sleep(0.1)
    sampler.stop()
    ms_t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if sharded:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_total = float(ms_t.item())
    ms_step = ms_total / args.steps

    F = U.kernel_model_flops(h, w, spec)
    value = F / (ms_step / 1e3) / 1e12
    peak = peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"])
    peak_sus = peaks.get("bf16_tflops_sustained", FALLBACK_PEAKS["bf16_tflops_sustained"])

    # ---- e2e through the public API with pinned host buffers.  Every step copies its input
    # host -> device and its result device -> host inside the timed region; consecutive steps are
    # pipelined on three streams (H2D of step i+1 and D2H of step i-1 overlap the compute of step i,
    # double-buffered device buffers), as a production caller streaming matrices would run it.
    e2e = None
    if not args.no_e2e:
        x_host = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        x_host.copy_(x)
        y_host = [torch.empty(y.shape, dtype=y.dtype, pin_memory=True) for _ in range(2)]
        xd = [torch.empty_like(x) for _ in range(2)]
        yd = [torch.empty_like(y) for _ in range(2)]
        s_h2d, s_cmp, s_d2h = (torch.cuda.Stream(device=dev) for _ in range(3))
        ev_h2d = [torch.cuda.Event() for _ in range(2)]
        ev_cmp = [torch.cuda.Event() for _ in range(2)]
        ev_d2h = [torch.cuda.Event() for _ in range(2)]
        started = [False, False]

        def e2e_step(i):
            j = i % 2
            with torch.cuda.stream(s_h2d):
                if started[j]:
                    s_h2d.wait_event(ev_cmp[j])      # step i-2 finished reading xd[j]
                xd[j].copy_(x_host, non_blocking=True)
                ev_h2d[j].record(s_h2d)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_h2d[j])
                if started[j]:
                    s_cmp.wait_event(ev_d2h[j])      # step i-2's result left yd[j]
                if not sharded:
                    U.orthogonalize(xd[j], spec, out=yd[j], check=False)
                else:
                    orthogonalize_row_sharded(xd[j], spec, out=yd[j], check=False, collective=args.collective)
                ev_cmp[j].record(s_cmp)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev_cmp[j])
                y_host[j].copy_(yd[j], non_blocking=True)
                ev_d2h[j].record(s_d2h)
            started[j] = True

        for i in range(2):
            e2e_step(i)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_h2d)
        for i in range(args.e2e_steps):
            e2e_step(i)
        s_d2h.wait_stream(s_cmp)
        e1.record(s_d2h)
        torch.cuda.synchronize()
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if sharded:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e_ms = float(et.item()) / args.e2e_steps
        nbytes = x.numel() * x.element_size()
        e2e = {"value": F / (e_ms / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": nbytes * world, "d2h_bytes_per_step": nbytes * world,
               "path": "pinned host -> device copy, unso_orthogonalize, device -> pinned host copy; "
                       "consecutive steps pipelined on three streams (double-buffered)"}

    # ---- roofline of the dominant kernel (stage times from CUDA events inside the timed region)
    roofline = None
    stages = None
    if stage_ms is not None and len(stage_ms):
        mean = stage_ms.mean(axis=0)
        stages = {n: float(v) for n, v in zip(N.PROFILE_STAGES, mean)}
        algo = {"gram": 2.0 * w * h * h, "apply": 2.0 * w * h * h,
                "chain": 2.0 * (spec.coeffs.order - 1) * h ** 3}
        dom = max(algo, key=lambda k: stages[k])
        achieved = algo[dom] / (stages[dom] / 1e3) / 1e12
        traffic = None
        tp = os.path.join(REPO, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            with open(tp) as fh:
                traffic = json.load(fh).get(f"{dom}:{rows}x{cols}:{args.precision}")
        roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "frac_of_sustained": achieved / peak_sus, "traffic": traffic,
                    "peak_source": f"{peaks_src} bf16_tflops (burst)",
                    "algorithmic_flops_per_launch": algo[dom], "avg_launch_ms": stages[dom]}

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        srows = min(args.cpu_sample_rows, rows)
        f, dt = cpu_oracle_sample(srows, cols, 99, bf16=args.precision == "bf16")
        cpu_base = {"value": f / dt / 1e12, "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "port",
                    "sample": f"one UNSO orthogonalization of a {srows}x{cols} row sample (fp64 numpy oracle)",
                    "seconds": dt}

    clocks = sampler.summary(t_wall0, t_wall1)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic: i.i.d. N(0,1) from torch.Generator(seed 1234+rank), no dataset",
            "config": {"workload": f"configs[3]: one {rows}x{cols} {args.precision} matrix, UNSO order-14 "
                                   "shipped coefficients", "global_batch": 1, "shape": [rows, cols],
                       "precision_recipe": ("bf16 Gram, bf16x3 C-form chain, "
                                            + {None: "adaptive bf16/bf16x2 (shifted P)", 1: "bf16", 2: "bf16x2"}[
                                                args.apply_terms] + " apply")
                       if args.precision == "bf16" else "fp64-grade DFMA",
                       "parallelism": (f"row-shard x{world} + " + ("NCCL all-reduce of G" if args.collective == "nccl" else
                                 "NVLink peer-memory reduction of G")) if sharded else "1 GPU",
                       "l2": "input 1 GiB > 126 MB L2 (no flush needed)"},
            "matrices_per_s": 1e3 / ms_step,
            "pct_bf16_peak": value / peak,
            "pct_bf16_peak_sustained": value / peak_sus,
            "flops_per_matrix": F,
            "roofline": roofline,
            "stages_ms": stages,
            "cpu_baseline": cpu_base,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "ortho_error": ortho_err,
            "ortho_error_reference": ortho_ref,
            "ortho_error_reference_how": "exact-arithmetic value of the reference polynomial on this input: "
                                         "sqrt(sum (g(sigma_i)^2 - 1)^2), sigma from the fp64 Gram of X",
            "apply_decision": None if apply_info is None else {
                "single_term": bool(apply_info["apply_single"]), "bound": apply_info["apply_bound"],
                "shift": apply_info["shift"]},
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
