"""The device epilogue sigmoid32 (common.cuh) against the reference's
(network.hpp:54-59, glibc exp in double).  Bit-exact except where CUDA's
double exp (<= 1 ulp) and glibc's differ in the last bit right at a float
rounding boundary; those are counted and bounded."""
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


def ulp_diff(a, b):
    return np.abs(a.view(np.int32).astype(np.int64) - b.view(np.int32).astype(np.int64))


def test_known_answers():
    y = dev_sigmoid(np.array([0.0, 0.5, 1.0, -1.0, 200.0, -200.0], np.float32))
    assert y[0] == np.float32(0.5)
    assert abs(float(y[1]) - 0.9230835512325638570) < 1e-7
    assert abs(float(y[2]) - 0.9931047268673538572) < 1e-7
    assert abs(float(y[3]) - 0.0068952731326461427) < 1e-9
    assert y[4].view(np.uint32) == np.float32(1.0 - 2.0 ** -24).view(np.uint32)
    assert y[5].view(np.uint32) == 1          # float denorm_min: no FTZ anywhere


def test_reference_golden():
    g = load_golden("sigmoid.npz")
    y = dev_sigmoid(g["x"])
    d = ulp_diff(y, g["y"])
    assert d.max() <= 1
    assert (d == 0).mean() >= 0.9999


def test_dense_sweep_against_oracle(oracle):
    rng = np.random.default_rng(5)
    x = np.concatenate([np.linspace(-20, 20, 1 << 22, dtype=np.float32),
                        rng.normal(0, 3, 1 << 22).astype(np.float32)])
    y = dev_sigmoid(x)
    r = oracle.sigmoid32(x)
    d = ulp_diff(y, r)
    assert d.max() <= 1
    mism = int((d != 0).sum())
    assert mism <= x.size * 1e-6, mism
