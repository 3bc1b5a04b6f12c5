#!/usr/bin/env python
"""UNSO orthogonalization benchmark on B200 (driver contract: one JSON line on rank 0).

Workloads (BASELINE.json configs, `--workload`, default cfg4):

  cfg4  configs[3]: one tall bf16 matrix 262144 x 2048, N(0,1).  The config the metric's 1/2/4/8-GPU
        figure and the north_star's >= 60 % of peak / >= 80 % scaling targets are quoted on.  N > 1:
        rows sharded along the long side, local Gram -> one all-reduce of the 2048 x 2048 Gram
        (NCCL, or --collective nvlink: the peer-memory reduction) -> redundant P(A) -> local apply
        (strong scaling).
  cfg1  configs[0]: one 512 x 128 fp32 matrix, N(0,1), fp32 mode (fp64-grade, parity <= 1e-5).
        Does not shard: N > 1 runs N replicas (weak scaling).
  cfg2  configs[1]: 16 x 2048 x 512 fp32, X = U diag(s) V^T, Haar U/V, s log-uniform [1e-4, 1];
        fp32 mode by default (--precision bf16 for the tensor-core mode).  N > 1: batch shares.
  cfg3  configs[2]: one Muon optimizer step (paper_2602_02500_b200.Muon: momentum, Nesterov, grouped
        orthogonalize, update) over 32 layers x {4 x 4096^2, 2 x 14336 x 4096, 4096 x 14336} bf16
        parameters, gradients N(0, 0.02^2).  N > 1: Muon(distribute=True) shares every shape group
        over the ranks and all-gathers the updates (strong scaling).
  cfg5  configs[4]: 4 x 16384 x 8192 fp32, Haar U/V, s = 1 + Pareto(1.5) min-max rescaled to
        [1e-6, 1]; bf16 mode by default, --precision fp32 for the fp64-grade mode.  N > 1: batch shares.

A step = one pass of the hot path over the workload's batch (cfg3: one optimizer step).
value    = reference-model FLOPs (kernel_model_flops, ortho.py:313-335) per second, whole job.
executed = the FLOPs the device actually issues (SYRK upper tiles, truncated chain, split products;
           e4m3 products counted at half a bf16 FLOP), and that rate as a fraction of the bf16 peak.
e2e      = the same metric through the public API from pinned host buffers: every step copies its
           input host -> device and its result device -> host inside the timed region.
--impl reference times the CPU oracle (numpy fp64 restatement of the reference, OpenBLAS on all
host threads) on a bounded sample of the workload; cpu_baseline in the ours arm times the SAME sample.

--gpus N > 1 without torchrun's environment re-launches this script under torch.distributed.run
with N ranks (one per GPU); under torchrun WORLD_SIZE must equal --gpus.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "UNSO orthogonalization TFLOP/s & matrices/s (% bf16 tensor peak), 1/2/4/8 B200"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
CPU_FULL_RECORD = os.path.join(REPO, "profiles", "cpu_full_workload.json")


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default per workload)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"], default="cfg4")
    ap.add_argument("--rows", type=int, default=None, help="cfg4: rows of the tall matrix (default 262144)")
    ap.add_argument("--cols", type=int, default=None, help="cfg4: columns (default 2048)")
    ap.add_argument("--layers", type=int, default=32, help="cfg3: transformer layers")
    ap.add_argument("--precision", choices=["bf16", "fp32"], default=None, help="default per workload")
    ap.add_argument("--collective", choices=["nccl", "nvlink"], default="nccl",
                    help="cfg4, N > 1: Gram all-reduce through NCCL, or the peer-memory reduction")
    ap.add_argument("--apply-terms", type=int, choices=[1, 2], default=None,
                    help="bf16 apply split: default adaptive per matrix (device-side bound)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-sample-rows", type=int, default=None,
                    help="cfg4: rows of the CPU sample timed by cpu_baseline AND --impl reference (default 32768)")
    ap.add_argument("--ref-sample-rows", type=int, default=None, help="alias of --cpu-sample-rows")
    ap.add_argument("--cpu-full", action="store_true",
                    help="also time the CPU oracle on the FULL workload once and record it in "
                         "profiles/cpu_full_workload.json (minutes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-projection", action="store_true", help="cfg4: skip the per-rank shard projection")
    ap.add_argument("--no-stage-profile", action="store_true",
                    help="developer A/B: do not record the library's per-stage CUDA events inside the timed "
                         "region (no stages_ms / roofline timing; shows what the ~7 event records per call cost)")
    ap.add_argument("--no-comparison", action="store_true",
                    help="skip the untimed-for-value NS comparison (5 Muon-coefficient steps, configs[0])")
    ap.add_argument("--sharded", action="store_true",
                    help="cfg4: run the row-sharded multi-rank path (process group, Gram reduction) even at world 1")
    ap.add_argument("--probe-ranks", action="store_true", help=argparse.SUPPRESS)  # launcher self-test (CPU)
    args = ap.parse_args(argv)
    if args.ref_sample_rows and not args.cpu_sample_rows:
        args.cpu_sample_rows = args.ref_sample_rows
    return args


# ----------------------------------------------------------------------------- launcher

def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_command(argv, gpus: int, port: int | None = None) -> list[str]:
    """The torch.distributed.run command that runs this script with `gpus` ranks on one node."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port or _free_port()),
            os.path.abspath(__file__), *argv]


def maybe_relaunch(args, argv) -> bool:
    """--gpus N > 1 outside torchrun: re-run under torch.distributed.run (N ranks) and return True.
    Under torchrun, WORLD_SIZE must match --gpus (a mismatch would silently report another N)."""
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None:
        if args.gpus > 1:
            rc = subprocess.call(launch_command(argv, args.gpus))
            sys.exit(rc)
        return False
    if int(world_env) != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world_env} but --gpus {args.gpus}; launch one rank per GPU")
    return False


def probe_ranks():
    """Launcher self-test: every rank joins a gloo group and rank 0 prints the ranks it saw."""
    import torch.distributed as dist
    dist.init_process_group("gloo")
    seen = [None] * dist.get_world_size()
    dist.all_gather_object(seen, {"rank": dist.get_rank(), "pid": os.getpid()})
    if dist.get_rank() == 0:
        print(json.dumps({"probe": True, "world": dist.get_world_size(), "ranks": seen}), flush=True)
    dist.destroy_process_group()


# ----------------------------------------------------------------------------- helpers

def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh), "measured"
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
                self.samples.append((time.time(), float(parts[0]), float(parts[1]), float(parts[2]), parts[3:7]))
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
        reasons = sorted({n for s in win for n, v in zip(self.NAMES, s[4]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(s[1] for s in win), "sm_max_mhz": max(s[2] for s in win),
                "power_w_max": max(s[3] for s in win), "reasons": reasons, "samples": len(win)}


def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("internal_api") in ("openblas", "mkl")]
        if n and n[0]:
            return int(n[0])
    except Exception:
        pass
    return os.cpu_count() or 1


# ----------------------------------------------------------------------------- CPU samples (oracle)
# The ONLY place (with --impl reference) where bench.py executes oracle/: the reported CPU baseline.

def cpu_sample_spec(args) -> dict:
    """The bounded CPU sample of each workload: the same one in cpu_baseline and --impl reference."""
    wl = args.workload
    if wl == "cfg4":
        rows, cols = _cfg4_shape(args)
        srows = min(args.cpu_sample_rows or 32768, rows)
        return {"method": "unso", "shapes": [(srows, cols)], "bf16": (args.precision or "bf16") == "bf16",
                "desc": f"one UNSO orthogonalization of a {srows}x{cols} row sample of the {rows}x{cols} workload "
                        f"(= one rank's shard at {max(rows // srows, 1)} GPUs)"}
    if wl == "cfg1":
        return {"method": "unso", "shapes": [(512, 128)], "bf16": False, "desc": "the full configs[0] matrix"}
    if wl == "cfg2":
        return {"method": "unso", "shapes": [(2048, 512)] * 4, "bf16": (args.precision or "fp32") == "bf16",
                "desc": "4 of the 16 configs[1] matrices (2048x512)"}
    if wl == "cfg3":
        return {"method": "unso", "shapes": [(4096, 4096)], "bf16": True,
                "desc": "one 4096x4096 of the 224 configs[2] matrices (orthogonalization only)"}
    return {"method": "unso", "shapes": [(16384, 4096)], "bf16": (args.precision or "bf16") == "bf16",
            "desc": "one 16384x4096 matrix (h = 4096 instead of configs[4]'s 8192: one full 16384x8192 "
                    "takes ~100 s on the host)"}


def cpu_oracle_run(spec: dict, seed: int):
    """Time the CPU oracle on the sample; returns (model FLOPs, seconds)."""
    import numpy as np
    import torch
    from oracle import unso_oracle as O
    flops, secs = 0, 0.0
    for i, (r, c) in enumerate(spec["shapes"]):
        g = torch.Generator().manual_seed(seed + i)
        m = torch.randn(r, c, generator=g)
        if spec["bf16"]:
            m = m.to(torch.bfloat16)
        m = np.ascontiguousarray(m.double().numpy())
        t0 = time.perf_counter()
        O.run(m, spec["method"])
        secs += time.perf_counter() - t0
        flops += O.model_flops(spec["method"], min(r, c), max(r, c))
    return flops, secs


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores, rank 0 only (other ranks exit 0)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    spec = cpu_sample_spec(args)
    steps = args.steps if args.steps is not None else 10
    for i in range(min(args.warmup, 1)):  # one untimed pass warms OpenBLAS' thread pool
        cpu_oracle_run(spec, 7 + i)
    fl, secs = 0, []
    for i in range(steps):
        f, dt = cpu_oracle_run(spec, 100 + i)
        fl = f
        secs.append(dt)
    total = sum(secs)
    value = fl * len(secs) / total / 1e12
    cores = cpu_threads()
    sample = f"{spec['desc']}; fp64 numpy/OpenBLAS oracle restating unso.ortho.orthogonalize; {steps} timed steps"
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(secs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_NAMES[args.workload] + f" (CPU sample: {spec['desc']})",
                   "parallelism": f"{cores} host threads"},
        "matrices_per_s": len(spec["shapes"]) * len(secs) / total,
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    rec = _cpu_full_record(args)
    if rec:
        line["cpu_baseline"]["full_workload_recorded"] = rec
    print(json.dumps(line), flush=True)


def _cpu_full_record(args):
    if not os.path.exists(CPU_FULL_RECORD):
        return None
    with open(CPU_FULL_RECORD) as fh:
        return json.load(fh).get(args.workload)


def cpu_full_measure(args):
    """--cpu-full: the CPU oracle on the FULL cfg4 matrix once (~100 s); recorded for later lines."""
    import numpy as np
    import torch
    from oracle import unso_oracle as O
    rows, cols = _cfg4_shape(args)
    g = torch.Generator().manual_seed(1234)
    m = np.ascontiguousarray(torch.randn(rows, cols, generator=g).to(torch.bfloat16).double().numpy())
    t0 = time.perf_counter()
    O.run(m, "unso")
    dt = time.perf_counter() - t0
    f = O.model_flops("unso", min(rows, cols), max(rows, cols))
    rec = {"value": f / dt / 1e12, "unit": "TFLOP/s", "seconds": dt, "cores": cpu_threads(), "kind": "port",
           "sample": f"the full {rows}x{cols} matrix, one UNSO orthogonalization",
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    data = {}
    if os.path.exists(CPU_FULL_RECORD):
        with open(CPU_FULL_RECORD) as fh:
            data = json.load(fh)
    data[args.workload] = rec
    with open(CPU_FULL_RECORD, "w") as fh:
        json.dump(data, fh, indent=1)
    return rec


# ----------------------------------------------------------------------------- executed-FLOP model

def _tiles(h: int, t: int) -> int:
    n = -(-h // t)
    return n * (n + 1) // 2


def executed_flops_bf16_unso(h: int, w: int, order: int, chain_steps: float, apply_single: bool,
                             route: str) -> dict:
    """FLOPs the bf16-mode UNSO kernels issue for one h x w matrix (bf16-equivalent: an e4m3 product
    costs half a bf16 product on tcgen05).  Mirrors the routes of csrc/unso_b200.cu:
      gram     CTA-pair SYRK, 256 x 256 upper tiles over the long side;
      chain    persistent (h <= 2048): 128 x 128 upper tiles, bf16x3 (3 products), chain_steps squarings
               (device-side truncation); glue-free (h > 2048): 256 x 256 pair tiles, squarings 1-3
               hi*hi (1 product), the rest hi*hi + two e4m3 cross terms (2 bf16-equivalents);
      apply    X (R_hi [+ R_lo]): 1 or 2 products of the full h x h P."""
    hp256 = -(-h // 256) * 256
    gram = 2.0 * w * 256 * 256 * _tiles(h, 256)
    if route == "persistent":
        hp = -(-h // 128) * 128
        chain = chain_steps * 3 * 2.0 * hp * 128 * 128 * _tiles(h, 128)
    else:
        per = 2.0 * hp256 * 256 * 256 * _tiles(h, 256)
        hi_only = 3 if order >= 12 else 0
        n = order - 1
        chain = per * (min(hi_only, n) + 2 * max(n - hi_only, 0))
    apply = 2.0 * w * h * h * (1 if apply_single else 2)
    return {"gram": gram, "chain": chain, "apply": apply, "total": gram + chain + apply}


OZ_BM, OZ_BN, OZ_PRODUCTS = 256, 96, 15  # csrc/ozaki_i8.cuh: CTA-pair tile, S(S+1)/2 digit products (S = 5)


def _oz_syrk_tiles(h: int) -> int:
    tm, tn = -(-h // OZ_BM), -(-h // OZ_BN)
    return sum(max(0, tn - (OZ_BM * i) // OZ_BN) for i in range(tm))


def executed_ops_int8_unso(h: int, w: int, order: int, tall: bool) -> dict:
    """int8 tensor-core ops (2 per MAC) the fp32-mode digit engine issues for one h x w matrix
    (csrc/ozaki_i8.cuh, h > 256): every contraction is 15 int8 products over 256 x 96 pair tiles --
    the Gram and each of the order-1 squarings as SYRKs (upper pair tiles), the apply over all tiles."""
    hp64 = -(-h // 64) * 64
    wp64 = -(-w // 64) * 64
    tile = 2.0 * OZ_BM * OZ_BN * OZ_PRODUCTS
    gram = tile * wp64 * _oz_syrk_tiles(h)
    chain = (order - 1) * tile * hp64 * _oz_syrk_tiles(h)
    m, n = (w, h) if tall else (h, w)
    apply = tile * hp64 * (-(-m // OZ_BM)) * (-(-n // OZ_BN))
    return {"gram": gram, "chain": chain, "apply": apply, "total": gram + chain + apply}


# ----------------------------------------------------------------------------- workloads

WORKLOAD_NAMES = {
    "cfg1": "configs[0]: one 512x128 fp32 matrix N(0,1), UNSO order-14",
    "cfg2": "configs[1]: 16 x 2048x512 fp32, Haar U/V, s log-uniform [1e-4,1], UNSO order-14",
    "cfg3": "configs[2]: Muon optimizer step, 32 layers x {4x 4096x4096, 2x 14336x4096, 4096x14336} bf16",
    "cfg4": "configs[3]: one 262144x2048 bf16 matrix N(0,1), UNSO order-14",
    "cfg5": "configs[4]: 4 x 16384x8192 fp32, Haar U/V, Pareto(1.5) spectrum in [1e-6,1], UNSO order-14",
}


def _cfg4_shape(args):
    return (args.rows or 262144), (args.cols or 2048)


def _controlled(batch, rows, cols, seeds, dev, spectrum):
    """X = U diag(s) V^T with Haar U (rows x k), V (cols x k) in fp64 on the device (seeded)."""
    import numpy as np
    import torch
    k = min(rows, cols)
    out = torch.empty(batch, rows, cols, dtype=torch.float32, device=dev)
    for b in range(batch):
        g = torch.Generator(device=dev).manual_seed(seeds[b])

        def haar(n):
            q, r = torch.linalg.qr(torch.randn(n, k, generator=g, device=dev, dtype=torch.float64))
            return q * torch.sign(torch.diagonal(r))
        s = torch.from_numpy(spectrum(np.random.default_rng(seeds[b]), k)).to(dev)
        out[b] = ((haar(rows) * s[None, :]) @ haar(cols).T).float()
        torch.cuda.synchronize(dev)
    return out


def _logu(rng, k):
    import numpy as np
    return np.exp(rng.uniform(np.log(1e-4), 0.0, k))


def _pareto(rng, k):
    s = 1.0 + rng.pareto(1.5, k)
    return 1e-6 + (s - s.min()) / (s.max() - s.min()) * (1.0 - 1e-6)


class MatrixWorkload:
    """One orthogonalize call per step over this rank's matrices (a 2-D matrix or a 3-D batch)."""

    def __init__(self, args, U, dev, rank, world):
        import torch
        self.args, self.U, self.dev, self.rank, self.world = args, U, dev, rank, world
        wl = args.workload
        self.sharded = False
        self.precision = args.precision or {"cfg1": "fp32", "cfg2": "fp32", "cfg4": "bf16", "cfg5": "bf16"}[wl]
        self.spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), precision=self.precision,
                                 apply_terms=args.apply_terms)
        if wl == "cfg4":
            rows, cols = _cfg4_shape(args)
            self.sharded = world > 1 or args.sharded
            from paper_2602_02500_b200.distributed import row_shard_bounds
            r0, r1 = row_shard_bounds(rows, world, rank) if self.sharded else (0, rows)
            g = torch.Generator(device=dev).manual_seed(1234 + rank)
            dt = torch.bfloat16 if self.precision == "bf16" else torch.float32
            self.x = torch.randn(r1 - r0, cols, generator=g, device=dev, dtype=torch.float32).to(dt)
            self.shape, self.total_batch, self.scaling = (rows, cols), 1, "strong"
            self.data = "synthetic: i.i.d. N(0,1) from torch.Generator(seed 1234+rank), no dataset"
        elif wl == "cfg1":
            g = torch.Generator(device=dev).manual_seed(0)
            self.x = torch.randn(512, 128, generator=g, device=dev, dtype=torch.float32)
            if self.precision == "bf16":
                self.x = self.x.to(torch.bfloat16)
            self.shape, self.total_batch, self.scaling = (512, 128), world, "weak"
            self.data = "synthetic: i.i.d. N(0,1) (torch.Generator seed 0); N > 1 = independent replicas"
        else:
            batch, rows, cols, spec_fn = ((16, 2048, 512, _logu) if wl == "cfg2" else (4, 16384, 8192, _pareto))
            per = -(-batch // world)
            mine = list(range(min(batch, rank * per), min(batch, (rank + 1) * per)))
            self.x = _controlled(len(mine), rows, cols, [11 + i for i in mine], dev, spec_fn) if mine else None
            if self.x is not None and self.precision == "bf16" and wl == "cfg2":
                pass  # fp32 input, bf16 mode: the library rounds it once (ortho: bf16 operand copy)
            self.shape, self.total_batch, self.scaling = (rows, cols), batch, "strong"
            self.data = ("synthetic: Haar U/V (QR of seeded Gaussians, fp64 on the device) x "
                         + ("log-uniform [1e-4,1]" if wl == "cfg2" else "Pareto(1.5) rescaled to [1e-6,1]")
                         + f" spectrum; {len(mine)} of {batch} matrices on this rank")
        rows, cols = self.shape
        self.h, self.w = (cols, rows) if rows > cols else (rows, cols)
        self.y = torch.empty_like(self.x) if self.x is not None else None
        self.model_flops = self.U.kernel_model_flops(self.h, self.w, self.spec) * self.total_batch
        self.launches = 0

    # the timed step
    def step(self, x=None, y=None):
        x = self.x if x is None else x
        y = self.y if y is None else y
        if x is None:
            return
        if self.sharded:
            from paper_2602_02500_b200.distributed import orthogonalize_row_sharded
            orthogonalize_row_sharded(x, self.spec, out=y, check=False, collective=self.args.collective)
        else:
            self.U.orthogonalize(x, self.spec, out=y, check=False)

    def gate(self):
        """Untimed: status check, our orthogonality error, the reference's exact-arithmetic value."""
        import numpy as np
        import torch
        import torch.distributed as dist
        U, N = self.U, self.U._native
        out = {"info": None}
        if self.x is None:
            return out
        if not self.sharded:
            res = U.orthogonalize(self.x, self.spec, out=self.y, check=True)
            self.launches = res.launches
            out["info"] = res.info
        else:
            from paper_2602_02500_b200 import distributed as D
            D.orthogonalize_row_sharded(self.x, self.spec, out=self.y, check=True, collective=self.args.collective)
            if self.args.collective == "nccl":
                g = D.native_gram(self.x, self.spec, None)
                self.launches = N.launch_count()
            else:
                red = D._nvlink_reducer(self.h, self.x.shape[0], None, self.dev)
                red.push(self.x, self.spec, None)
                self.launches = N.launch_count()
                red.reduce()
                self.launches += N.launch_count()
                g = red.wait()
                self.launches += N.launch_count()
            D.native_finish(self.x, g, self.spec, None, self.y)
            self.launches += N.launch_count()
        torch.cuda.synchronize()
        ys = self.y if self.y.dim() == 3 else self.y[None]
        xs = self.x if self.x.dim() == 3 else self.x[None]
        errs, refs = [], []
        for b in range(ys.shape[0]):
            yf, xf = ys[b].double(), xs[b].double()
            tall = yf.shape[0] > yf.shape[1]
            gy = yf.T @ yf if tall else yf @ yf.T
            gx = xf.T @ xf if tall else xf @ xf.T
            if self.sharded:
                dist.all_reduce(gy)
                dist.all_reduce(gx)
            errs.append(float(torch.linalg.norm(gy - torch.eye(gy.shape[0], device=gy.device, dtype=gy.dtype))))
            # the reference's result has singular values g(sigma(X)/s) (scalar_map, ortho.py:286-310)
            sx = torch.sqrt(torch.linalg.eigvalsh(gx).clamp_min(0.0)).cpu().numpy()
            sy = U.scalar_map(self.spec)(sx / float((sx ** 4).sum()) ** 0.25)
            refs.append(float(np.sqrt(((sy ** 2 - 1.0) ** 2).sum())))
        out["ortho_error"] = errs[0] if len(errs) == 1 else errs
        out["ortho_error_reference"] = refs[0] if len(refs) == 1 else refs
        return out

    def executed(self, info):
        """Executed bf16-equivalent FLOPs per step (whole job) in bf16 mode; int8 tensor-core ops of
        the digit engine in fp32 mode (h > 256)."""
        if self.precision == "fp32" and self.h > 256:
            e = executed_ops_int8_unso(self.h, self.w, self.spec.coeffs.order, self.shape[0] > self.shape[1])
            e = {k: v * self.total_batch for k, v in e.items()}
            e["unit"] = "int8 ops"
            return e
        if self.precision != "bf16" or not info:
            return None
        route = "persistent" if self.h <= 2048 else "glue-free"
        tot = {"gram": 0.0, "chain": 0.0, "apply": 0.0, "total": 0.0}
        for d in info:
            e = executed_flops_bf16_unso(self.h, self.w, self.spec.coeffs.order, d["chain_steps"] or 13,
                                         bool(d["apply_single"]), route)
            for k in tot:
                tot[k] += e[k] * (self.total_batch / len(info))
        return tot

    def stage_model(self):
        """Algorithmic (model) FLOPs per call of each stage, this rank."""
        b = 1 if self.x is None or self.x.dim() == 2 else self.x.shape[0]
        h, w = self.h, (self.x.shape[-2] if self.sharded else self.w)
        return {"gram": 2.0 * w * h * h * b, "apply": 2.0 * w * h * h * b,
                "chain": 2.0 * (self.spec.coeffs.order - 1) * h ** 3 * b}

    def hbm_bytes(self):
        """Algorithmic HBM bytes of the stand-alone reduction/normalisation stages (per call):
        finalize_p reads the fp32 P upper triangle and writes P/s - dI as bf16 hi + lo (both triangles)."""
        b = 1 if self.x is None or self.x.dim() == 2 else self.x.shape[0]
        return {"finalize_p": 6.0 * self.h * self.h * b}

    def host_io(self):
        return [self.x], [self.y]


class MuonWorkload:
    """configs[2]: one Muon optimizer step over the synthetic layer stack (bf16)."""

    SHAPES = [(4096, 4096)] * 4 + [(14336, 4096)] * 2 + [(4096, 14336)]

    def __init__(self, args, U, dev, rank, world):
        import torch
        self.args, self.U, self.dev, self.rank, self.world = args, U, dev, rank, world
        self.precision = args.precision or "bf16"
        self.sharded = world > 1
        g = torch.Generator(device=dev).manual_seed(7)  # same on every rank: replicated (all-reduced) grads
        self.params = []
        for _ in range(args.layers):
            for s in self.SHAPES:
                p = torch.nn.Parameter(torch.zeros(s, dtype=torch.bfloat16, device=dev))
                p.grad = (torch.randn(s, generator=g, device=dev) * 0.02).to(torch.bfloat16)
                self.params.append(p)
        self.opt = U.Muon(self.params, lr=0.02, momentum=0.95, precision=self.precision, distribute=self.sharded)
        self.spec = self.opt.spec
        self.model_flops = sum(U.kernel_model_flops(min(p.shape), max(p.shape), self.spec) for p in self.params)
        self.total_batch = len(self.params)
        self.scaling = "strong"
        self.shape = None
        self.data = ("synthetic: bf16 parameters (zeros) with gradients i.i.d. N(0, 0.02^2) from "
                     "torch.Generator(seed 7), identical on every rank (as after a data-parallel all-reduce)")
        self.launches = 0

    def step(self):
        self.opt.step()

    def gate(self):
        """Untimed: orthogonality errors of one matrix of each shape group, and the call structure."""
        import numpy as np
        import torch
        U, N = self.U, self.U._native
        out = {"info": {}}
        errs, refs = {}, {}
        launches = 2 * 3  # the fused momentum/prepare and update passes of the 3 shape groups
        for s in sorted(set(self.SHAPES)):
            items = [p for p in self.params if tuple(p.shape) == s]
            stacked = torch.stack([p.grad for p in items[: max(1, len(items) // self.world)]])
            res = U.orthogonalize(stacked, self.spec, precision=self.precision, check=True)
            launches += res.launches
            out["info"][f"{s[0]}x{s[1]}"] = res.info
            y, x = res.y[0].double(), stacked[0].double()
            tall = y.shape[0] > y.shape[1]
            gy = y.T @ y if tall else y @ y.T
            gx = x.T @ x if tall else x @ x.T
            errs[f"{s[0]}x{s[1]}"] = float(torch.linalg.norm(gy - torch.eye(gy.shape[0], device=gy.device,
                                                                            dtype=gy.dtype)))
            sx = torch.sqrt(torch.linalg.eigvalsh(gx).clamp_min(0.0)).cpu().numpy()
            sy = U.scalar_map(self.spec)(sx / float((sx ** 4).sum()) ** 0.25)
            refs[f"{s[0]}x{s[1]}"] = float(np.sqrt(((sy ** 2 - 1.0) ** 2).sum()))
        self.launches = launches
        self.opt.step()  # allocates the momentum buffers before timing
        torch.cuda.synchronize()
        out["ortho_error"] = errs
        out["ortho_error_reference"] = refs
        return out

    def executed(self, info):
        if self.precision != "bf16" or not info:
            return None
        tot = {"gram": 0.0, "chain": 0.0, "apply": 0.0, "total": 0.0}
        for key, rows in info.items():
            r, c = map(int, key.split("x"))
            h, w = min(r, c), max(r, c)
            n = sum(1 for p in self.params if tuple(p.shape) == (r, c))
            for d in rows:
                e = executed_flops_bf16_unso(h, w, self.spec.coeffs.order, d["chain_steps"] or 13,
                                             bool(d["apply_single"]), "persistent" if h <= 2048 else "glue-free")
                for k in tot:
                    tot[k] += e[k] * n / len(rows)
        return tot

    def stage_model(self):
        """Model FLOPs per step of each stage, summed over the groups (this rank's share)."""
        tot = {"gram": 0.0, "apply": 0.0, "chain": 0.0}
        for p in self.params:
            h, w = min(p.shape), max(p.shape)
            tot["gram"] += 2.0 * w * h * h / self.world
            tot["apply"] += 2.0 * w * h * h / self.world
            tot["chain"] += 2.0 * (self.spec.coeffs.order - 1) * h ** 3 / self.world
        return tot

    def hbm_bytes(self):
        return {"finalize_p": sum(6.0 * min(p.shape) ** 2 for p in self.params) / self.world}


# ----------------------------------------------------------------------------- e2e

def run_e2e_matrix(work, steps, dev):
    """Pinned host -> device copy of each step's input, the public API call, device -> pinned host
    copy of the result; consecutive steps pipelined on three streams (double-buffered)."""
    import torch
    if work.x is None:
        return None
    x, y = work.x, work.y
    x_host = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    x_host.copy_(x)
    y_host = [torch.empty(y.shape, dtype=y.dtype, pin_memory=True) for _ in range(2)]
    xd = [torch.empty_like(x) for _ in range(2)]
    yd = [torch.empty_like(y) for _ in range(2)]
    s_h2d, s_cmp, s_d2h = (torch.cuda.Stream(device=dev) for _ in range(3))
    ev_cmp = [torch.cuda.Event() for _ in range(2)]
    ev_h2d = [torch.cuda.Event() for _ in range(2)]
    ev_d2h = [torch.cuda.Event() for _ in range(2)]
    started = [False, False]

    def e2e_step(i):
        j = i % 2
        with torch.cuda.stream(s_h2d):
            if started[j]:
                s_h2d.wait_event(ev_cmp[j])
            xd[j].copy_(x_host, non_blocking=True)
            ev_h2d[j].record(s_h2d)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev_h2d[j])
            if started[j]:
                s_cmp.wait_event(ev_d2h[j])
            work.step(xd[j], yd[j])
            ev_cmp[j].record(s_cmp)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev_cmp[j])
            y_host[j].copy_(yd[j], non_blocking=True)
            ev_d2h[j].record(s_d2h)
        started[j] = True

    for i in range(2):
        e2e_step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_h2d)
    for i in range(steps):
        e2e_step(i)
    s_d2h.wait_stream(s_cmp)
    e1.record(s_d2h)
    torch.cuda.synchronize()
    nbytes = x.numel() * x.element_size()
    return e0.elapsed_time(e1) / steps, nbytes, y.numel() * y.element_size(), (
        "pinned host -> device copy, orthogonalize (unso_orthogonalize), device -> pinned host copy; consecutive "
        "steps pipelined on three streams (double-buffered)")


def run_e2e_muon(work, steps, dev):
    """Gradients copied in from pinned host memory, the optimizer step, the updated parameters copied
    back to pinned host memory, every step -- pipelined by shape group: one Muon instance per group
    (the same per-group work as the single optimizer of the headline step), the H2D copy of group g+1
    and the D2H copy of group g-1 overlapping the step of group g on three streams."""
    import torch
    U = work.U
    U.ortho.workspace_pool.clear()  # the headline step's workspace (default stream) makes room for the
    torch.cuda.empty_cache()        # compute stream's (workspaces are per stream; ~64 GB for a 4096² group)
    groups = {}
    for p in work.params:
        groups.setdefault(tuple(p.shape), []).append(p)
    opts = [U.Muon(ps, lr=0.02, momentum=0.95, precision=work.precision, distribute=work.sharded)
            for ps in groups.values()]
    plist = [ps for ps in groups.values()]
    grads_h = [[torch.empty(p.shape, dtype=p.dtype, pin_memory=True) for p in ps] for ps in plist]
    params_h = [[torch.empty(p.shape, dtype=p.dtype, pin_memory=True) for p in ps] for ps in plist]
    for ghs, ps in zip(grads_h, plist):
        for gh, p in zip(ghs, ps):
            gh.copy_(p.grad)
    s_h2d, s_cmp, s_d2h = (torch.cuda.Stream(device=dev) for _ in range(3))
    ng = len(plist)
    ev_h2d = [torch.cuda.Event() for _ in range(ng)]
    ev_cmp = [torch.cuda.Event() for _ in range(ng)]
    ev_d2h = [torch.cuda.Event() for _ in range(ng)]
    started = [False] * ng

    def one_step():
        for g in range(ng):
            with torch.cuda.stream(s_h2d):
                if started[g]:
                    s_h2d.wait_event(ev_cmp[g])  # the previous step's group g consumed its gradients
                for gh, p in zip(grads_h[g], plist[g]):
                    p.grad.copy_(gh, non_blocking=True)
                ev_h2d[g].record(s_h2d)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_h2d[g])
                if started[g]:
                    s_cmp.wait_event(ev_d2h[g])  # parameters read back before they are updated again
                opts[g].step()
                ev_cmp[g].record(s_cmp)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev_cmp[g])
                for ph, p in zip(params_h[g], plist[g]):
                    ph.copy_(p.detach(), non_blocking=True)
                ev_d2h[g].record(s_d2h)
            started[g] = True

    one_step()  # warm-up (allocations, pointer lists)
    torch.cuda.synchronize()
    if os.environ.get("UNSO_BENCH_E2E_TRACE"):  # developer: per-group timeline of two pipelined steps (stderr)
        tr = []
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(s_h2d)
        for st in range(2):
            for g in range(ng):
                marks = {}
                for name, strm in (("h2d", s_h2d), ("cmp", s_cmp), ("d2h", s_d2h)):
                    marks[name] = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                with torch.cuda.stream(s_h2d):
                    s_h2d.wait_event(ev_cmp[g])
                    marks["h2d"][0].record(s_h2d)
                    for gh, p in zip(grads_h[g], plist[g]):
                        p.grad.copy_(gh, non_blocking=True)
                    marks["h2d"][1].record(s_h2d)
                    ev_h2d[g].record(s_h2d)
                with torch.cuda.stream(s_cmp):
                    s_cmp.wait_event(ev_h2d[g])
                    s_cmp.wait_event(ev_d2h[g])
                    marks["cmp"][0].record(s_cmp)
                    opts[g].step()
                    marks["cmp"][1].record(s_cmp)
                    ev_cmp[g].record(s_cmp)
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(ev_cmp[g])
                    marks["d2h"][0].record(s_d2h)
                    for ph, p in zip(params_h[g], plist[g]):
                        ph.copy_(p.detach(), non_blocking=True)
                    marks["d2h"][1].record(s_d2h)
                    ev_d2h[g].record(s_d2h)
                tr.append((st, g, marks))
        torch.cuda.synchronize()
        for st, g, marks in tr:
            print(f"[e2e trace] step {st} group {g} ({len(plist[g])} x {tuple(plist[g][0].shape)}): " + ", ".join(
                f"{k} {t0.elapsed_time(a):.0f}-{t0.elapsed_time(b):.0f} ms" for k, (a, b) in marks.items()),
                file=sys.stderr)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    done = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    e0.record(s_h2d)
    for i in range(steps):
        one_step()
        done[i].record(s_d2h)  # the step's last parameters are back on the host
    s_d2h.wait_stream(s_cmp)
    s_d2h.wait_stream(s_h2d)
    e1.record(s_d2h)
    torch.cuda.synchronize()
    nbytes = sum(p.numel() * p.element_size() for p in work.params)
    how = ("gradients pinned host -> device, Muon.step per shape group (grouped orthogonalize), updated "
           "parameters device -> pinned host; the copies of neighbouring groups overlap each group's step "
           "on three streams")
    if steps > 1:  # whole-run average includes the pipeline's fill (first H2D) and drain (last D2H)
        steady = done[0].elapsed_time(done[-1]) / (steps - 1)
        how += f"; steady state (completion to completion of consecutive steps): {steady:.1f} ms per step"
    return e0.elapsed_time(e1) / steps, nbytes, nbytes, how


def recorded_chain_phases(h, hbm_peak):
    """The reduction / normalisation phases of configs[3] run inside the persistent chain kernel, so the
    stage events cannot time them; this reports their durations from the committed phase timeline of
    the timing build (tools/chain_trace.py -> profiles/round2_end_chain_trace_cfg4.txt; a recorded
    figure, not measured in this run) against their algorithmic bytes (L2-resident data)."""
    path = os.path.join(REPO, "profiles", "round2_end_chain_trace_cfg4.txt")
    out = {"source": "profiles/round2_end_chain_trace_cfg4.txt (timing build, recorded; not measured in this run)"}
    try:
        import re
        line = next(ln for ln in open(path) if "phase A:" in ln)
        us_a = float(re.search(r"partials\+norms ([0-9.]+) us", line).group(1))
        us_p = float(re.search(r"P split\+mirror ([0-9.]+)", line).group(1))
    except Exception:  # noqa: BLE001
        return None
    nt = (h + 127) // 128
    tiles = nt * (nt + 1) // 2
    splits = 2
    a_bytes = tiles * 128 * 128 * 4 * splits                # split-K fp32 Gram partials in (upper tiles)
    p_bytes = h * h * 2 * 2                                 # P/s as bf16 hi + lo, both triangles, out
    out["split_k_sum_and_norms"] = {"bytes": a_bytes, "us": us_a, "GB/s": a_bytes / us_a / 1e3,
                                    "frac_of_hbm_peak": a_bytes / us_a / 1e3 / hbm_peak}
    out["p_split_and_mirror"] = {"bytes": p_bytes, "us": us_p, "GB/s": p_bytes / us_p / 1e3,
                                 "frac_of_hbm_peak": p_bytes / us_p / 1e3 / hbm_peak}
    return out


# ----------------------------------------------------------------------------- main

def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    args = parse_args(argv)
    if args.probe_ranks:
        if not maybe_relaunch(args, argv):
            probe_ranks()
        return
    if args.impl == "reference":
        if os.environ.get("WORLD_SIZE") is None or int(os.environ.get("RANK", "0")) == 0:
            run_reference(args)
        return
    maybe_relaunch(args, argv)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2602_02500_b200 as U
    from paper_2602_02500_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    multi = world > 1 or args.sharded
    if multi:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if multi:
            dist.barrier()

    wl = args.workload
    steps = args.steps if args.steps is not None else {"cfg1": 200, "cfg2": 50, "cfg3": 3, "cfg4": 50,
                                                       "cfg5": 5}[wl]
    if wl == "cfg3" and args.precision == "fp32":
        sys.exit("bench.py: cfg3 runs in bf16 mode")
    work = MuonWorkload(args, U, dev, rank, world) if wl == "cfg3" else MatrixWorkload(args, U, dev, rank, world)
    gate = work.gate()

    for _ in range(max(args.warmup, 0)):
        work.step()
    torch.cuda.synchronize()
    barrier()

    peaks, peaks_src = load_peaks()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    stream = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    calls_per_step = 3 if wl == "cfg3" else 1
    want_prof = world == 1 and not args.sharded and not args.no_stage_profile
    # The library's stage events (~7 cudaEventRecord per call) cost nothing measurable on the large
    # workloads but 5-20 % on the latency-bound configs[0] / configs[1] (A/B with --no-stage-profile):
    # those time `value` without them and take the stage breakdown from a second pass of the same steps.
    two_pass = want_prof and wl in ("cfg1", "cfg2")
    prof = N.StageProfiler(steps * calls_per_step) if (want_prof and not two_pass) else None
    if prof:
        prof.__enter__()
    barrier()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    ev0.record(stream)
    for _ in range(steps):
        work.step()
    ev1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.time()
    barrier()
    ms_local = ev0.elapsed_time(ev1)
    stage_ms = prof.read() if prof else None
    if prof:
        prof.__exit__(None, None, None)
    ms_profiled = None
    if two_pass:
        with N.StageProfiler(steps * calls_per_step) as prof2:
            torch.cuda.synchronize()
            ev0.record(stream)  # ms_local was read above
            for _ in range(steps):
                work.step()
            ev1.record(stream)
            torch.cuda.synchronize()
            ms_profiled = ev0.elapsed_time(ev1) / steps
            stage_ms = prof2.read()
    time.sleep(0.1)
    sampler.stop()
    ms_t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if multi:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_step = float(ms_t.item()) / steps

    F = work.model_flops
    value = F / (ms_step / 1e3) / 1e12
    peak = peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"])
    peak_sus = peaks.get("bf16_tflops_sustained", FALLBACK_PEAKS["bf16_tflops_sustained"])
    hbm_peak = peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])

    # ---- executed work (what the tensor cores actually issue)
    execd = work.executed(gate.get("info"))
    executed = None
    int8_peak = 2.0 * peak  # B200 dense int8 = 2x dense bf16 (4.5 POPS vs 2.25 PFLOPS); no measured int8 peak
    if execd and execd.get("unit") == "int8 ops":
        executed = {"int8_ops_per_step": execd["total"], "tops": execd["total"] / (ms_step / 1e3) / 1e12,
                    "frac_of_int8_peak": execd["total"] / (ms_step / 1e3) / 1e12 / int8_peak,
                    "by_stage": {k: execd[k] for k in ("gram", "chain", "apply")},
                    "int8_peak_tops": int8_peak,
                    "how": "int8 tcgen05.mma ops the fp32-mode digit engine issues (15 digit products per "
                           "contraction, 256 x 96 pair tiles, SYRK upper tiles); int8 peak = 2 x the measured "
                           "bf16 burst peak (datasheet ratio)"}
    elif execd:
        executed = {"flops_per_step": execd["total"], "tflops": execd["total"] / (ms_step / 1e3) / 1e12,
                    "frac_of_peak": execd["total"] / (ms_step / 1e3) / 1e12 / peak,
                    "by_stage": {k: execd[k] for k in ("gram", "chain", "apply")},
                    "how": "bf16-equivalent FLOPs the kernels issue: SYRK upper tiles, truncated chain, "
                           "split products (e4m3 at half a bf16 FLOP)"}

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e_steps = args.e2e_steps or (4 if wl == "cfg3" else min(30, max(steps, 4)))  # cfg3: ~0.55 s per step
        barrier()
        r = run_e2e_muon(work, e_steps, dev) if wl == "cfg3" else run_e2e_matrix(work, e_steps, dev)
        if r is not None:
            e_ms, bi, bo, path = r
        else:
            e_ms, bi, bo, path = 0.0, 0, 0, "no matrices on this rank"
        et = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        bt = torch.tensor([bi, bo], dtype=torch.float64, device=dev)
        if multi:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
            dist.all_reduce(bt)
        e_ms = float(et.item())
        e2e = {"value": F / (e_ms / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(bt[0].item()), "d2h_bytes_per_step": int(bt[1].item()), "path": path}

    # ---- roofline of the dominant kernel (stage times from CUDA events inside the timed region)
    roofline, stages, hbm = None, None, None
    if stage_ms is not None and len(stage_ms):
        per_step = stage_ms.reshape(steps, calls_per_step, -1).sum(axis=1).mean(axis=0)
        stages = {n: float(v) for n, v in zip(N.PROFILE_STAGES, per_step)}
        algo = work.stage_model()
        dom = max(algo, key=lambda k: stages[k])
        achieved = algo[dom] / (stages[dom] / 1e3) / 1e12
        traffic = None
        tp = os.path.join(REPO, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            with open(tp) as fh:
                traffic = json.load(fh).get(f"{dom}:{wl}:{work.precision}")
        roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "frac_of_sustained": achieved / peak_sus, "traffic": traffic,
                    "peak_source": f"{peaks_src} bf16_tflops (burst)",
                    "algorithmic_flops_per_step": algo[dom], "stage_ms_per_step": stages[dom]}
        if execd and execd.get("unit") == "int8 ops" and dom in execd:
            # fp32 mode: the dominant contraction runs on the int8 tensor cores -- its roofline is int8 ops
            ach = execd[dom] / (stages[dom] / 1e3) / 1e12
            roofline.update({"achieved": ach, "peak": int8_peak, "unit": "TOPS (int8)", "frac": ach / int8_peak,
                             "frac_of_sustained": ach / (2.0 * peak_sus),
                             "peak_source": f"2 x {peaks_src} bf16_tflops (burst): dense int8 = 2x bf16",
                             "algorithmic_int8_ops_per_step": execd[dom],
                             "model_tflops_fp64_equivalent": algo[dom] / (stages[dom] / 1e3) / 1e12})
        elif execd and dom in execd:
            roofline["executed_tflops"] = execd[dom] / (stages[dom] / 1e3) / 1e12
            roofline["executed_frac"] = roofline["executed_tflops"] / peak
        hb = work.hbm_bytes()
        hbm = {}
        for k, nbytes in hb.items():
            if stages.get(k, 0.0) > 0.01:  # a stand-alone stage (fused into the chain kernel otherwise)
                gbs = nbytes / (stages[k] / 1e3) / 1e9
                hbm[k] = {"bytes_per_step": nbytes, "ms_per_step": stages[k], "GB/s": gbs, "frac": gbs / hbm_peak}
            else:
                hbm[k] = {"fused": "into the persistent chain kernel (no stand-alone launch)",
                          "ms_per_step": stages.get(k)}
        if wl == "cfg4" and work.h == 2048 and work.precision == "bf16":
            hbm["chain_phases_recorded"] = recorded_chain_phases(work.h, hbm_peak)

    # ---- cfg4: per-rank critical path of an N-way row shard, measured on this GPU
    projection = None
    if wl == "cfg4" and world == 1 and not args.sharded and not args.no_projection:
        projection = shard_projection(work, U, N, dev, ms_step)

    # ---- the NS comparison path (configs[0]: "compared against 5 Muon-coefficient NS steps")
    comparison = None
    if (wl != "cfg3" and world == 1 and not args.sharded and not args.no_comparison
            and not (wl == "cfg5" and work.precision == "fp32")):
        comparison = ns_comparison(work, U, dev, ms_step, {"cfg1": 50, "cfg2": 10, "cfg4": 5, "cfg5": 2}[wl])

    # ---- CPU baseline: the same bounded sample as --impl reference, on this box's host cores
    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        spec = cpu_sample_spec(args)
        f, dt = cpu_oracle_run(spec, 100)
        cpu_base = {"value": f / dt / 1e12, "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "port",
                    "sample": spec["desc"] + " (fp64 numpy oracle; same sample as --impl reference)",
                    "seconds": dt}
        rec = cpu_full_measure(args) if (args.cpu_full and wl == "cfg4") else _cpu_full_record(args)
        if rec:
            cpu_base["full_workload_recorded"] = rec

    clocks = sampler.summary(t_wall0, t_wall1)
    if rank == 0:
        shape = work.shape
        cfg = {"workload": WORKLOAD_NAMES[wl] + ("" if args.rows is None and args.cols is None else
                                                f" (shape overridden: {shape[0]}x{shape[1]})"),
               "global_batch": work.total_batch,
               "precision_mode": work.precision,
               "parallelism": parallelism_name(wl, world, multi, args.collective),
               "l2": "inputs larger than the 126 MB L2 (no flush needed)" if wl in ("cfg3", "cfg4", "cfg5") else
                     "working set fits in L2: inputs stay L2-resident between steps (latency-bound config)"}
        if shape:
            cfg["shape"] = list(shape)
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": work.scaling, "vs_baseline": None, "dtype": work.precision,
            "data": work.data, "config": cfg,
            "matrices_per_s": work.total_batch / (ms_step / 1e3),
            "model_flops_per_step": F,
            "pct_bf16_peak_model_flops": value / peak,
            "executed": executed,
            "roofline": roofline,
            "hbm_stages": hbm,
            "stages_ms": stages,
            "stage_profile": ({"pass": "second pass of the same steps (stage events cost 5-20 % on this latency-bound "
                                       "config, so the timed pass runs without them)",
                               "ms_per_step_with_stage_events": ms_profiled}
                              if two_pass else {"pass": "timed region"} if stage_ms is not None else None),
            "cpu_baseline": cpu_base,
            "e2e": e2e,
            "gpu_launches": work.launches * steps if work.launches else None,
            "clocks": clocks,
            "ortho_error": gate.get("ortho_error"),
            "ortho_error_reference": gate.get("ortho_error_reference"),
            "ortho_error_reference_how": "exact-arithmetic value of the reference polynomial on this input: "
                                         "sqrt(sum (g(sigma_i)^2 - 1)^2), sigma from the fp64 Gram of X",
        }
        if projection:
            line["shard_projection"] = projection
        if comparison:
            line["comparison"] = comparison
        info = gate.get("info")
        if isinstance(info, list) and info and wl == "cfg4":
            d = info[0]
            line["apply_decision"] = {"single_term": bool(d["apply_single"]), "bound": d["apply_bound"],
                                      "shift": d["shift"], "chain_steps": d["chain_steps"]}
        print(json.dumps(line), flush=True)
    if multi:
        dist.destroy_process_group()


def ns_comparison(work, U, dev, ms_unso, steps):
    """The comparison path of configs[0] (and of the other matrix configs): 5 Muon-coefficient NS steps
    (ortho.py:221-237) on the same input and precision, timed like the headline (CUDA events, inputs
    resident); its orthogonality error next to the reference's exact-arithmetic value (the composed
    quintic map on sigma(X)/||X||_F, plain scaling)."""
    import numpy as np
    import torch
    spec_m = U.MethodSpec(U.MethodKind.MUON_NS, iterations=5)
    yc = torch.empty_like(work.x)
    for _ in range(2):
        U.orthogonalize(work.x, spec_m, precision=work.precision, out=yc, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        U.orthogonalize(work.x, spec_m, precision=work.precision, out=yc, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    F = U.kernel_model_flops(work.h, work.w, spec_m) * work.total_batch
    y0 = (yc if yc.dim() == 2 else yc[0]).double()
    x0 = (work.x if work.x.dim() == 2 else work.x[0]).double()
    tall = y0.shape[0] > y0.shape[1]
    gy = y0.T @ y0 if tall else y0 @ y0.T
    gx = x0.T @ x0 if tall else x0 @ x0.T
    err = float(torch.linalg.norm(gy - torch.eye(gy.shape[0], device=gy.device, dtype=gy.dtype)))
    sx = torch.sqrt(torch.linalg.eigvalsh(gx).clamp_min(0.0)).cpu().numpy()
    sy = U.scalar_map(spec_m)(sx / float(np.sqrt((sx ** 2).sum())))
    return {"method": "Muon-5 Newton-Schulz, (a,b,c) = (3.4445, -4.7750, 2.0315) x 5, plain scaling",
            "ms_per_step": ms, "model_flops_per_step": F, "model_tflops": F / (ms / 1e3) / 1e12,
            "unso_speedup": ms / ms_unso, "steps": steps,
            "ortho_error": err, "ortho_error_reference": float(np.sqrt(((sy ** 2 - 1.0) ** 2).sum()))}


def parallelism_name(wl, world, multi, collective):
    if not multi:
        return "1 GPU"
    if wl == "cfg4":
        return f"row-shard x{world} + " + ("NCCL all-reduce of G" if collective == "nccl" else
                                           "NVLink peer-memory reduction of G")
    if wl == "cfg1":
        return f"{world} independent replicas"
    if wl == "cfg3":
        return f"data-parallel Muon: shape-group shares x{world} + all-gather of the updates"
    return f"batch shares x{world}, no communication"


def shard_projection(work, U, N, dev, ms_full):
    """Measured per-rank critical path of the row-sharded cfg4 at N = 2, 4, 8 on this one GPU: one
    rank's stages on its w/N rows exactly as orthogonalize_row_sharded runs them -- the local Gram
    (unso_gram), then scale + chain + apply from the GLOBAL Gram (unso_orthogonalize_from_gram; the
    all-reduce's result is stood in for by the full matrix's Gram, so the scale, truncation and apply
    decision are the full problem's) -- timed with CUDA events, plus an ASSUMED Gram all-reduce
    (not measurable on one GPU: 16.8 MB fp32, 700 GB/s bus bandwidth + 15 us latency).
    Projected efficiency = T_1 / (N * T_N)."""
    import torch
    from paper_2602_02500_b200 import distributed as D
    out = {}
    rows = work.x.shape[0]
    h = work.h
    g_full = D.native_gram(work.x, work.spec, None)
    ar_bytes = 4.0 * h * h
    for n in (2, 4, 8):
        xs = work.x[: rows // n]
        ys = torch.empty_like(xs)
        gbuf = torch.empty_like(g_full)
        reps = 20
        t_g, t_f = 0.0, 0.0
        for it in range(reps + 3):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            g = D.native_gram(xs, work.spec, None)
            e1.record()
            gbuf.copy_(g_full)  # the all-reduce's result (not timed; the all-reduce is assumed below)
            e2.record()
            D.native_finish(xs, gbuf, work.spec, None, ys)
            e3 = torch.cuda.Event(enable_timing=True)
            e3.record()
            torch.cuda.synchronize()
            del g
            if it >= 3:
                t_g += e0.elapsed_time(e1) / reps
                t_f += e2.elapsed_time(e3) / reps
        t_ar = 1e3 * (2.0 * (n - 1) / n * ar_bytes / 700e9) + 0.015
        t_n = t_g + t_f + t_ar
        # the same two stages replayed as CUDA graphs: the GPU-side critical path without the host
        # launch gaps of ~0.1 ms stages (a rank would capture gram -> all-reduce -> finish the same way)
        t_gg = t_fg = None
        try:
            gg, gf = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                for _ in range(2):  # warm-up on the capture stream (workspace, attributes)
                    D.native_gram(xs, work.spec, None)
                    D.native_finish(xs, gbuf, work.spec, None, ys)
                with torch.cuda.graph(gg, stream=side):
                    D.native_gram(xs, work.spec, None)
                with torch.cuda.graph(gf, stream=side):
                    D.native_finish(xs, gbuf, work.spec, None, ys)
            torch.cuda.current_stream(dev).wait_stream(side)
            torch.cuda.synchronize()
            for graph, key in ((gg, "g"), (gf, "f")):
                graph.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    graph.replay()
                e1.record()
                torch.cuda.synchronize()
                if key == "g":
                    t_gg = e0.elapsed_time(e1) / reps
                else:
                    t_fg = e0.elapsed_time(e1) / reps
        except Exception as exc:  # graph capture unavailable: report the event-timed path only
            print(f"bench.py: graphed shard projection skipped: {exc}", file=sys.stderr)
        rec = {"rows_per_rank": rows // n, "gram_ms": t_g, "chain_and_apply_ms": t_f,
               "allreduce_ms_assumed": t_ar, "critical_path_ms": t_n,
               "projected_efficiency": ms_full / (n * t_n)}
        if t_gg is not None and t_fg is not None:
            t_ng = t_gg + t_fg + t_ar
            rec.update({"gram_ms_graphed": t_gg, "chain_and_apply_ms_graphed": t_fg,
                        "critical_path_ms_graphed": t_ng, "projected_efficiency_graphed": ms_full / (n * t_ng)})
        out[str(n)] = rec
    return out


if __name__ == "__main__":
    main()
