"""Batches on the persistent bf16 chain's two-slot form (chain_persistent.cuh): a chunk that one
wave of CTAs cannot hold runs as two matrix groups, slot s of every CTA in group s, each group with
its own barrier rounds and its own data-dependent truncation decision (ortho.py:197-204 is the
reference: all N - 1 squarings, per matrix).

Covered here against the CPU oracle, matrix by matrix:
  * groups of equal and unequal size (odd batches), CTAs with one and with two slots in one launch,
  * one group truncating early (tall well-conditioned inputs) while the other runs all squarings
    (ill-conditioned inputs), in both orders, and matrices of both kinds inside one group
    (the group then runs to the slowest matrix),
  * several chunks (batch larger than two waves) and h = 2048 batches (136 tiles per matrix: one
    matrix per group),
  * ragged h (padding rows / columns of the last tile row) in a two-group launch.
Bar: relative Frobenius error <= 2e-2 per matrix (bf16 mode), every output finite."""

import numpy as np
import pytest
import torch

import paper_2602_02500_b200 as U
from oracle import unso_oracle as O

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
UNSO = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
TOL = 2e-2


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def well_conditioned(w, h, seed):
    """Tall Gaussian: sigma within a few percent of each other, the chain truncates early."""
    g = torch.Generator(device=DEV).manual_seed(seed)
    return torch.randn(w, h, generator=g, device=DEV)


def ill_conditioned(w, h, seed):
    """Haar U, V with sigma log-uniform in [1e-4, 1]: every squaring runs."""
    rng = np.random.default_rng(seed)
    s = np.exp(rng.uniform(np.log(1e-4), 0.0, size=h))
    return torch.from_numpy(O.controlled_spectrum_matrix(w, h, s, seed)).to(DEV, torch.float32)


def run_and_check(mats, label):
    x = torch.stack(mats).to(torch.bfloat16)
    res = U.orthogonalize(x, UNSO, precision="bf16")
    torch.cuda.synchronize()
    y = res.y
    assert torch.isfinite(y).all(), label
    worst = 0.0
    for i in range(x.shape[0]):
        ref = O.run(x[i].double().cpu().numpy(), "unso")["y"]
        r = rel(y[i].double().cpu().numpy(), ref)
        worst = max(worst, r)
        assert r <= TOL + 2.0 ** -9, (label, i, r)
    steps = [int(d["chain_steps"]) for d in res.info] if isinstance(res.info, list) else None
    print(f"{label}: worst rel err vs oracle {worst:.2e}, chain steps per matrix {steps}")
    return steps


@pytest.mark.parametrize("order", ["trunc_first", "trunc_second", "mixed"])
def test_groups_with_different_truncation(order):
    """16 x (2048 x 512): 160 tiles -> two groups of 8 matrices on 80 CTAs."""
    w, h, nb = 2048, 512, 16
    good = [well_conditioned(w, h, 100 + i) for i in range(nb // 2)]
    bad = [ill_conditioned(w, h, 200 + i) for i in range(nb // 2)]
    if order == "trunc_first":
        mats = good + bad
    elif order == "trunc_second":
        mats = bad + good
    else:
        mats = [m for pair in zip(good, bad) for m in pair]
    steps = run_and_check(mats, f"h=512 batch 16 {order}")
    if steps is not None and order != "mixed":
        lo, hi = (steps[:8], steps[8:]) if order == "trunc_first" else (steps[8:], steps[:8])
        assert max(lo) < min(hi), steps  # the well-conditioned group stopped earlier than the other one


@pytest.mark.parametrize("shape,nb", [((1536, 512), 15), ((1536, 512), 17), ((2304, 1024), 5), ((1024, 384), 31),
                                      ((1200, 500), 16), ((3000, 2048), 2), ((2500, 2048), 3),
                                      ((2100, 1990), 2), ((1024, 512), 61)])
def test_group_sizes_and_chunks(shape, nb):
    """Odd batches (unequal groups, CTAs with one and two slots), ragged h, several chunks,
    one 136-tile matrix per group."""
    w, h = shape
    mats = [(well_conditioned if i % 3 else ill_conditioned)(w, h, 1000 * h + 7 * nb + i) for i in range(nb)]
    run_and_check(mats, f"{w}x{h} batch {nb}")


def test_two_slot_matches_one_slot_per_matrix():
    """The same matrices orthogonalized one by one (one wave, one slot per CTA) and as a 16-batch (two
    groups): per-matrix results agree to bf16-mode accuracy (the truncation decision is per group,
    so the batch may run more squarings on a matrix than its own launch does)."""
    w, h, nb = 2048, 512, 16
    mats = [(well_conditioned if i % 2 else ill_conditioned)(w, h, 31 + i).to(torch.bfloat16) for i in range(nb)]
    yb = U.orthogonalize(torch.stack(mats), UNSO, precision="bf16").y
    torch.cuda.synchronize()
    for i, m in enumerate(mats):
        y1 = U.orthogonalize(m, UNSO, precision="bf16").y
        r = rel(yb[i].double().cpu().numpy(), y1.double().cpu().numpy())
        assert r <= 1e-2, (i, r)


@pytest.mark.parametrize("variant", ["plain", "no_truncation", "two_term_apply"])
def test_two_group_launch_with_spec_variants(variant):
    """The same two-group launch under the other recipe knobs of the path: plain (trace) scaling
    (ortho.py:153-154), the truncation switched off (every group runs all 13 squarings) and the forced
    bf16x2 apply."""
    w, h, nb = 1536, 512, 16
    kw = {"plain": dict(scaling="plain"), "no_truncation": dict(truncate=False),
          "two_term_apply": dict(apply_terms=2)}[variant]
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), **kw)
    mats = [(well_conditioned if i % 2 else ill_conditioned)(w, h, 77 + i) for i in range(nb)]
    x = torch.stack(mats).to(torch.bfloat16)
    res = U.orthogonalize(x, spec, precision="bf16")
    torch.cuda.synchronize()
    assert torch.isfinite(res.y).all()
    steps = [int(d["chain_steps"]) for d in res.info]
    if variant == "no_truncation":
        assert steps == [13] * nb, steps
    for i in range(nb):
        ref = O.run(x[i].double().cpu().numpy(), "unso", scaling="plain" if variant == "plain" else None)["y"]
        r = rel(res.y[i].double().cpu().numpy(), ref)
        assert r <= TOL + 2.0 ** -9, (variant, i, r)
