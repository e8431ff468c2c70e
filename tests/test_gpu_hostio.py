"""Host-buffer activation paths of asnn_dev_activate (eval_parallel +
read_outputs, eval.cpp:49-87): pageable buffers are staged with copies,
page-locked ones are read / written in place by the sweep's kernels
(zero-copy; K-cta writes the declared outputs itself).  All must give the
reference's values bit for bit."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2005_04347_b200 as A
from conftest import bitwise_equal

pytestmark = pytest.mark.gpu


def pinned_activate(dl, X: np.ndarray, n_vec: int, n_out: int) -> np.ndarray:
    x = torch.from_numpy(np.ascontiguousarray(X, np.float32).reshape(-1)).pin_memory()
    out = torch.full((n_out * n_vec,), -7.0, dtype=torch.float32).pin_memory()
    dl.activate_host_ptr(x.data_ptr(), n_vec, x.numel(), out.data_ptr())
    return out.numpy().copy()


@pytest.mark.parametrize("n_vec", [1, 16, 100, 128, 300])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_population_outputs_staged_and_zero_copy(oracle, n_vec, mode):
    rng = A.SplitMix64(91 + n_vec)
    nets = [A.generate(A.GenSpec(8, 4, 188, 1000, 8, seed=rng.next())) for _ in range(40)]
    pop = A.DeviceLayout.from_population(nets)
    dev = A.Device.get(0)
    dev.set_sweep_mode(mode)
    try:
        X = np.random.default_rng(n_vec).uniform(-2, 2, (40, n_vec, 8)).astype(np.float32)
        staged, _ = pop.activate(X, outputs=True, state=False, n_vec=n_vec)
        zc = pinned_activate(pop, X, n_vec, 40 * 4)
    finally:
        dev.set_sweep_mode(0)
    want = np.concatenate([oracle.eval_batch(oracle.layout(net), X[g])[:, net.outputs].reshape(-1)
                           for g, net in enumerate(nets)])
    assert bitwise_equal(staged.reshape(-1), want)
    assert bitwise_equal(zc, want)


@pytest.mark.parametrize("n_vec", [1, 64, 200])
def test_single_network_zero_copy(oracle, n_vec):
    net = A.generate_powerlaw(5000, 12, 32, 16, 100_000, 2.1, 3)
    d = oracle.layout(net)
    dl = A.DeviceLayout.from_network(net)
    X = np.random.default_rng(7).uniform(-2, 2, (n_vec, len(net.inputs))).astype(np.float32)
    zc = pinned_activate(dl, X, n_vec, len(net.outputs))
    staged, _ = dl.activate(X, outputs=True)
    want = oracle.eval_batch(d, X)[:, net.outputs].reshape(-1)
    assert bitwise_equal(staged.reshape(-1), want)
    assert bitwise_equal(zc, want)
