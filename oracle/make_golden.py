"""Generate ``tests/golden/`` from the LIVE reference (build container only).

Run:  python oracle/make_golden.py

Imports the unmodified reference package from ``/root/reference/pkg/src``
(read-only; no install) and records its outputs on seeded inputs, then
cross-checks the numpy restatement in ``oracle/unso_oracle.py`` against the
same outputs.  ``/root/reference`` does not exist on the GPU box, so the GPU
tests consume only the committed fixtures written here.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")

sys.path.insert(0, REPO)
sys.dont_write_bytecode = True


def _ref():
    if not os.path.isdir(REF_SRC):
        raise SystemExit(f"reference not found at {REF_SRC}; fixtures are generated in the build container")
    sys.path.insert(0, REF_SRC)
    import unso  # noqa: F401  (the live reference)
    from unso import bench, ortho, rng, scalarpoly
    from unso.coeff_train import CesistaStepParams
    from unso.data import default_cesista_triples, default_coefficients
    return dict(unso=unso, bench=bench, ortho=ortho, rng=rng, scalarpoly=scalarpoly,
                CesistaStepParams=CesistaStepParams, default_coefficients=default_coefficients,
                default_cesista_triples=default_cesista_triples)


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64 (what the GPU sees)."""
    f = np.asarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = ((f + 0x7FFF + ((f >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32).astype(np.float64)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    R = _ref()
    ortho, scalarpoly, bench, rng = R["ortho"], R["scalarpoly"], R["bench"], R["rng"]
    from oracle import unso_oracle as O

    os.makedirs(OUT, exist_ok=True)
    coeffs = R["default_coefficients"]()
    assert coeffs.order == O.DEFAULT_ORDER and coeffs.b_rule.value == O.DEFAULT_RULE
    assert np.array_equal(coeffs.a, np.array(O.DEFAULT_A)), "vendored default coefficients drifted"
    ces_rows = R["default_cesista_triples"]()
    assert np.array_equal(np.asarray(ces_rows), np.array(O.CESISTA_DEFAULT_TRIPLES))
    ces = R["CesistaStepParams"](ces_rows)

    kat = {}
    # --- PRNG: words/uniforms/normals (rng.py) --------------------------------
    kat["rng_words_seed0"] = [int(v) for v in rng.raw_words(0, 0, 8)]
    kat["rng_words_seed7_start5"] = [int(v) for v in rng.raw_words(7, 5, 4)]
    kat["rng_normals_seed3"] = [float(v) for v in rng.normals(3, 0, 7)]
    g = bench.gaussian_matrix(512, 128, 0)
    kat["cfg1_input_sha256"] = sha(g)
    kat["cfg1_input_sum"] = float(g.sum())
    # --- coefficients (scalarpoly.py) -----------------------------------------
    kat["derive_b_default"] = scalarpoly.derive_b(coeffs)
    kat["derive_b_exact_n1"] = scalarpoly.derive_b(scalarpoly.CoefficientSet(1, np.zeros(0), "exact"))
    kat["derive_b_approxsum_n14_zero"] = scalarpoly.derive_b(
        scalarpoly.CoefficientSet(14, np.zeros(13), "approx-sum"))
    gen_a = (0.25 + rng.uniforms(17, 0, 13)).tolist()
    kat["generic_a"] = gen_a
    kat["derive_b_generic_abs"] = scalarpoly.derive_b(scalarpoly.CoefficientSet(14, np.array(gen_a), "approx-abs"))
    grid = np.linspace(0.0005, 1.0, 64)
    kat["eval_f_grid"] = grid.tolist()
    kat["eval_f_default"] = scalarpoly.eval_f(coeffs, grid).tolist()
    # --- scalar maps ------------------------------------------------------------
    specs = {
        "unso": ortho.MethodSpec(ortho.MethodKind.UNSO, coeffs=coeffs),
        "original8": ortho.MethodSpec(ortho.MethodKind.ORIGINAL_NS),
        "muon5": ortho.MethodSpec(ortho.MethodKind.MUON_NS),
        "cesista": ortho.MethodSpec(ortho.MethodKind.CESISTA_NS, step_params=ces),
    }
    kat["scalar_maps"] = {k: ortho.scalar_map(s)(grid).tolist() for k, s in specs.items()}
    # --- FLOP model -------------------------------------------------------------
    kat["flops"] = {}
    for (h, w) in [(128, 128), (128, 512), (128, 1024), (512, 2048), (2048, 262144), (4096, 4096),
                   (4096, 14336), (8192, 16384)]:
        kat["flops"][f"{h}x{w}"] = {k: int(ortho.kernel_model_flops(h, w, s)) for k, s in specs.items()}

    # --- small matrices: every method, ragged/tall/wide/square ------------------
    gen = scalarpoly.CoefficientSet(14, np.array(gen_a), "approx-abs")
    small_specs = {
        "unso_default": ortho.MethodSpec(ortho.MethodKind.UNSO, coeffs=coeffs),
        "unso_generic": ortho.MethodSpec(ortho.MethodKind.UNSO, coeffs=gen),
        "unso_plain": ortho.MethodSpec(ortho.MethodKind.UNSO, coeffs=coeffs, scaling="plain"),
        "unso_gelfand": ortho.MethodSpec(ortho.MethodKind.UNSO, coeffs=coeffs, scaling="gelfand"),
        "original4": ortho.MethodSpec(ortho.MethodKind.ORIGINAL_NS, iterations=4),
        "muon3": ortho.MethodSpec(ortho.MethodKind.MUON_NS, iterations=3),
        "muon5": ortho.MethodSpec(ortho.MethodKind.MUON_NS, iterations=5),
        "cesista": ortho.MethodSpec(ortho.MethodKind.CESISTA_NS, step_params=ces),
        "external": ortho.MethodSpec(ortho.MethodKind.EXTERNAL_SCHEDULE,
                                     schedule=np.tile(np.array(ortho.MUON_COEFFICIENTS), (3, 1))),
    }
    arrays = {}
    cases = []
    shapes = [(16, 40), (40, 16), (24, 24), (7, 13), (130, 66), (64, 256)]
    for (r, c) in shapes:
        m = bench.gaussian_matrix(r, c, r * 1000 + c)
        arrays[f"in_{r}x{c}"] = m
        for name, spec in small_specs.items():
            res = ortho.orthogonalize(m, spec)
            key = f"{name}_{r}x{c}"
            arrays[f"y_{key}"] = res.y
            cases.append(dict(key=key, input=f"in_{r}x{c}", method=name, flops=int(res.flops),
                              preprocess_flops=int(res.preprocess_flops),
                              was_transposed=bool(res.was_transposed),
                              shapes=[list(s) for s in res.kernel_matmul_shapes],
                              ortho_error=float(bench.ortho_error_any(res.y))))

    # --- cfg1 (512x128 fp32 from seed 0) and its bf16-rounded twin -------------
    m32 = np.asarray(g, dtype=np.float32).astype(np.float64)
    mbf = bf16_round(g)
    cfg1 = {}
    for tag, m in (("fp32", m32), ("bf16", mbf)):
        for name, spec in (("unso", specs["unso"]), ("muon5", specs["muon5"])):
            res = ortho.orthogonalize(m, spec)
            arrays[f"cfg1_{tag}_{name}"] = res.y
            cfg1[f"{tag}_{name}"] = dict(flops=int(res.flops), preprocess_flops=int(res.preprocess_flops),
                                         ortho_error=float(bench.ortho_error_any(res.y)),
                                         fro=float(np.linalg.norm(res.y)))

    # --- controlled spectrum (cfg2-like, reduced) ------------------------------
    s = np.exp(np.random.default_rng(11).uniform(np.log(1e-4), 0.0, 64))
    spec_in = O.controlled_spectrum_matrix(256, 64, s, 11)
    arrays["in_spectrum_256x64"] = spec_in
    arrays["s_spectrum_256x64"] = s
    res = ortho.orthogonalize(spec_in, specs["unso"])
    arrays["y_spectrum_256x64_unso"] = res.y
    res = ortho.orthogonalize(spec_in, specs["muon5"])
    arrays["y_spectrum_256x64_muon5"] = res.y

    np.savez_compressed(os.path.join(OUT, "reference_outputs.npz"), **arrays)
    with open(os.path.join(OUT, "reference_kats.json"), "w") as fh:
        json.dump(dict(kat=kat, cases=cases, cfg1=cfg1), fh, indent=1, sort_keys=True)

    # --- cross-check the restatement ---------------------------------------------
    worst = 0.0
    assert np.array_equal(O.gaussian_matrix(512, 128, 0), g), "rng restatement is not bit-exact"
    for case in cases:
        m = arrays[case["input"]]
        name = case["method"]
        kw = dict(unso_default=dict(method="unso"),
                  unso_generic=dict(method="unso", a=gen_a, rule="approx-abs"),
                  unso_plain=dict(method="unso", scaling="plain"),
                  unso_gelfand=dict(method="unso", scaling="gelfand"),
                  original4=dict(method="original", iterations=4),
                  muon3=dict(method="muon", iterations=3),
                  muon5=dict(method="muon", iterations=5),
                  cesista=dict(method="cesista", rows=O.cesista_rows(O.CESISTA_DEFAULT_TRIPLES)),
                  external=dict(method="external", rows=O.muon_rows(3)))[name]
        out = O.run(m, **kw)
        worst = max(worst, float(np.max(np.abs(out["y"] - arrays[f"y_{case['key']}"]))))
        assert out["flops"] == case["flops"], case["key"]
        assert out["preprocess_flops"] == case["preprocess_flops"], case["key"]
        assert [list(x) for x in out["shapes"]] == case["shapes"], case["key"]
    print(f"oracle vs live reference: max |dy| over {len(cases)} small cases = {worst:.3e}")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
