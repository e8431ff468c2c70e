"""The C-ABI library loads and exports every symbol include/asnn_dev.h
declares; without a GPU the device handle reports BackendUnavailable
(eval.cpp:51-52 semantics) instead of computing anything.  CPU only."""
from __future__ import annotations

import ctypes as C
import re

import pytest

from conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "asnn_dev.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(asnn_(?:dev|gen|corpus)_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("asnn_dev_open", "asnn_dev_compute_required", "asnn_dev_segment",
              "asnn_dev_build_layout", "asnn_dev_upload_layout", "asnn_dev_activate",
              "asnn_dev_layer_slice", "asnn_dev_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2005_04347_b200 import _lib
    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes prototype table covers them all
    assert set(declared_symbols()) <= set(_lib.PROTOTYPES)


def test_library_links_no_host_evaluator():
    """The product .so must not carry an evaluator of its own on the host:
    only the CUDA path and the corpus generators."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_2005_04347_b200" /
                                                             "libasnn_b200.so")],
                         capture_output=True, text=True, check=True).stdout
    assert "orc_" not in out and "eval_sequential" not in out


def test_no_gpu_is_backend_unavailable():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2005_04347_b200 import _lib
    import paper_2005_04347_b200 as A
    lib = _lib.load()
    h = C.c_void_p()
    assert lib.asnn_dev_open(0, C.byref(h)) == _lib.ASNN_E_UNAVAILABLE
    with pytest.raises(A.BackendUnavailable):
        A.Device(0)
    net = A.make_network([0, 1], [2], [(0, 2, 0.5), (1, 2, -0.25)])
    with pytest.raises(A.BackendUnavailable):
        A.compute_required(net)


def test_host_backend_is_not_silently_served():
    import numpy as np
    import paper_2005_04347_b200 as A
    lay = A.LayeredLayout(2, [0, 2, 3], [0, 1, 2], [0, 0, 0, 2], [0, 1], [0.5, -0.25], [0, 1], 0, 3)
    with pytest.raises(A.BackendUnavailable):
        A.eval_parallel(lay, np.zeros(2, np.float32), A.ParallelConfig())
    cfg = A.ParallelConfig(backend=A.Backend.DeviceCompute, node_hook=lambda i: None)
    with pytest.raises(A.BackendUnavailable):
        A.eval_parallel(lay, np.zeros(2, np.float32), cfg)
    with pytest.raises(A.InputArityMismatch):
        A.eval_parallel(lay, np.zeros(3, np.float32), A.ParallelConfig(backend=A.Backend.DeviceCompute))
