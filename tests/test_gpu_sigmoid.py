"""The device epilogue sigmoid32 (common.cuh, with the glibc exp restatement
of exp_glibc.h) against the reference's (network.hpp:54-59, glibc exp in
double): bit-exact, for the golden values, dense sweeps and -- exhaustively --
all 2^32 float inputs, compared with the reference's own sigmoid32 running on
this box's host libm."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import paper_2005_04347_b200 as A
from paper_2005_04347_b200 import _lib
from conftest import load_golden

pytestmark = pytest.mark.gpu


def dev_sigmoid(x):
    dev = A.Device.get(0)
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    dev.check(dev.lib.asnn_dev_sigmoid32(dev.h, _lib.ptr(x, C.c_float), _lib.ptr(y, C.c_float),
                                         x.size))
    return y


def test_known_answers():
    y = dev_sigmoid(np.array([0.0, 0.5, 1.0, -1.0, 200.0, -200.0], np.float32))
    assert y[0] == np.float32(0.5)
    assert abs(float(y[1]) - 0.9230835512325638570) < 1e-7
    assert abs(float(y[2]) - 0.9931047268673538572) < 1e-7
    assert abs(float(y[3]) - 0.0068952731326461427) < 1e-9
    assert y[4].view(np.uint32) == np.float32(1.0 - 2.0 ** -24).view(np.uint32)
    assert y[5].view(np.uint32) == 1          # float denorm_min: no FTZ anywhere


def test_reference_golden_bitwise():
    g = load_golden("sigmoid.npz")
    y = dev_sigmoid(g["x"])
    assert np.array_equal(y.view(np.uint32), g["y"].view(np.uint32))


def test_dense_sweep_bitwise(oracle):
    rng = np.random.default_rng(5)
    x = np.concatenate([np.linspace(-20, 20, 1 << 22, dtype=np.float32),
                        rng.normal(0, 3, 1 << 22).astype(np.float32)])
    assert np.array_equal(dev_sigmoid(x).view(np.uint32), oracle.sigmoid32(x).view(np.uint32))


def test_all_2pow32_inputs_bitwise(ref):
    """Every float bit pattern (NaNs included: both sides must agree on the
    bits of whatever they return) through the device and through the
    reference's sigmoid32 (oracle/_ref, OpenMP over the host cores)."""
    chunk = 1 << 28
    mism = 0
    for c in range(1 << 32 >> 28):
        bits = np.arange(c * chunk, (c + 1) * chunk, dtype=np.uint64).astype(np.uint32)
        x = bits.view(np.float32)
        d = dev_sigmoid(x).view(np.uint32)
        r = ref.sigmoid32(x).view(np.uint32)
        nan = np.isnan(x)
        mism += int(np.count_nonzero((d != r) & ~nan))
        assert np.all(np.isnan(d.view(np.float32)[nan]) == np.isnan(r.view(np.float32)[nan]))
    assert mism == 0


def test_fast_path_against_exact_all_inputs():
    """sigmoid32's fast path + rounding test (common.cuh) against the exact
    restatement for every float bit pattern, on the device."""
    dev = A.Device.get(0)
    bad, slow = C.c_uint64(), C.c_uint64()
    dev.check(dev.lib.asnn_dev_sigmoid_selfcheck(dev.h, C.byref(bad), C.byref(slow)))
    assert bad.value == 0
    # NaNs, the saturated tails and the rare near-midpoint values take the exact path
    assert slow.value < (1 << 32) // 4
