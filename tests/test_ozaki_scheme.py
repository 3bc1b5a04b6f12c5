"""CPU pins of the fp32 mode's int8 digit scheme (csrc/ozaki_i8.cuh), through its exact numpy
emulation (tools/ozaki_emulation.py: int8 digit products summed exactly, as the int8 tensor cores do):
the digits fit int8 (|d| <= 64), a group's int32 accumulator cannot overflow at the engine's K bound,
5 digits per operand keep the whole UNSO pipeline within the fp32-mode bar (1e-5) of the oracle on a
configs[1]-like spectrum, and 4 digits in the chain do not (the reason S = 5)."""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import unso_oracle as O  # noqa: E402
from tools import ozaki_emulation as Z  # noqa: E402


def test_digits_fit_int8_and_reconstruct():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((64, 300)) * np.exp2(rng.integers(-30, 30, (64, 1)))
    a[3] = 0.0
    e, digs = Z.split_rows(a, 5)
    assert max(np.max(np.abs(d)) for d in digs) <= 64
    rec = sum(d * 2.0 ** (-6 - 7 * s) for s, d in enumerate(digs)) * np.exp2(e)[:, None]
    scale = np.max(np.abs(a), axis=1, keepdims=True) + 1e-300
    assert np.max(np.abs(rec - a) / scale) <= 2.0 ** -(6 + 7 * 4)


def test_int32_accumulator_bound_at_max_k():
    # a group (s + t = g) holds at most S = 5 products of |d_s d_t| <= 64 * 64 summed over K
    assert 5 * 64 * 64 * 65536 < 2 ** 31  # OZ_MAX_K = 65536 per split-K slice


def test_five_digits_meet_the_fp32_bar_four_in_the_chain_do_not():
    rng = np.random.default_rng(3)
    s = np.exp(rng.uniform(np.log(1e-4), 0.0, 96))
    m = O.controlled_spectrum_matrix(384, 96, s, 5).astype(np.float32).astype(np.float64)
    ref = O.run(m, "unso")["y"].T  # the emulation works in the h x w orientation
    err5 = np.linalg.norm(Z.unso_ozaki(m, 5, 5, 5) - ref) / np.linalg.norm(ref)
    err4 = np.linalg.norm(Z.unso_ozaki(m, 5, 4, 5) - ref) / np.linalg.norm(ref)
    assert err5 <= 1e-6, err5
    assert err4 > 1e-5, err4  # 4 chain digits: 1.2e-5, over the fp32-mode bar
