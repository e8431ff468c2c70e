"""the bench corpora generated on the GPU (csrc/gen.cu).

Both generators are counter-based per node (csrc/gen_core.h, compiled into
the host generators in netgen.cpp and the device kernels in gen.cu), so the
device must reproduce the host networks byte for byte: node list, declared
inputs / outputs, every (source, target) pair in order and every weight's
bits.  At config 4's full size the generated-on-device network is levelled
and flattened on the device without touching the host, and must still equal
the reference's own preprocessing and activations (tests/golden/
fullsize_c4.npz, written by the unmodified reference)."""
from __future__ import annotations

import hashlib
import pathlib

import numpy as np
import pytest

import paper_2005_04347_b200 as A

pytestmark = pytest.mark.gpu


def same_network(a, b):
    for k in ("nodes", "inputs", "outputs", "source", "target"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert np.array_equal(a.weight.view(np.uint32), b.weight.view(np.uint32))


@pytest.mark.parametrize("layers,width,p,seed", [(3, 7, 0.5, 1), (12, 300, 0.1, 3), (40, 500, 0.02, 9),
                                                 (6, 64, 1.0, 2)])
def test_mlp_device_equals_host(layers, width, p, seed):
    same_network(A.device_generate_mlp(layers, width, p, seed), A.generate_mlp(layers, width, p, seed))


@pytest.mark.parametrize("args", [(20000, 10, 64, 32, 400000, 2.1, 5),      # test_corpus.py's shape
                                  (3000, 6, 16, 8, 300000, 1.6, 7),        # dense draws (k >= avail/2)
                                  (200_000, 40, 512, 512, 10_000_000, 2.1, 7),
                                  (1_000_000, 100, 1024, 1024, 50_000_000, 2.1, 4)])
def test_powerlaw_device_equals_host(args):
    same_network(A.device_generate_powerlaw(*args), A.generate_powerlaw(*args))


@pytest.mark.slow
def test_config4_generated_and_levelled_on_device():
    """Config 4 (495M edges) generated, levelled and flattened on the GPU:
    the layout hashes like the reference's segment / flatten of the host
    corpus, and the sweep of the fixture's 64 vectors like its eval_parallel."""
    import importlib.util
    path = pathlib.Path(__file__).resolve().parent / "golden" / "make_fullsize.py"
    spec = importlib.util.spec_from_file_location("make_fullsize", path)
    fx = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(fx)
    g = np.load(pathlib.Path(__file__).resolve().parent / "golden" / "fullsize_c4.npz")
    dl = A.DeviceLayout.generated_powerlaw(10_000_000, 100, 1024, 1024, 500_000_000, 2.1, 4)
    lay = dl.download()
    assert fx.layout_digest(dict(layer_offsets=lay.layer_offsets, node_ids=lay.node_ids,
                                 row_ptr=lay.row_ptr, in_nodes=lay.in_nodes, in_weights=lay.in_weights,
                                 input_order=lay.input_order)) == str(g["layout_sha256"])
    del lay
    out, st = dl.activate(g["x"], outputs=True, state=True)
    assert np.array_equal(out.view(np.uint32), g["outputs"].view(np.uint32))
    assert [fx.state_digest(s) for s in st] == [str(h) for h in g["state_sha256"]]
    dl.free()
