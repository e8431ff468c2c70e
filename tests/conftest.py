"""Shared fixtures.  `-m gpu` tests need a B200 and call through the C-ABI;
everything else runs on CPU (oracle, golden vectors, host logic, symbol
exports, gloo world_size-2 sharding)."""
from __future__ import annotations

import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: large shapes")


def split(arr: np.ndarray, lens: np.ndarray):
    out, k = [], 0
    for n in lens:
        out.append(arr[k:k + int(n)])
        k += int(n)
    return out


def load_golden(name: str) -> dict:
    return dict(np.load(GOLDEN / name))


@pytest.fixture(scope="session")
def oracle():
    from oracle.bind import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.bind import Ref, available_ref
    if not available_ref():
        pytest.skip("oracle/_ref not built (reference checkout absent at build time)")
    return Ref()


@pytest.fixture(scope="session")
def adversarial_nets():
    """The adversarial golden networks with the reference's answers."""
    import paper_2005_04347_b200 as A
    d = load_golden("adversarial.npz")
    cols = {k: split(d[k], d[k + "_len"]) for k in
            ("nodes", "inputs", "outputs", "source", "target", "weight", "required", "level",
             "flatten_ok", "x", "op", "dropped")}
    nets = []
    for i in range(len(cols["nodes"])):
        net = A.Network(cols["nodes"][i], cols["inputs"][i], cols["outputs"][i], cols["source"][i],
                        cols["target"][i], cols["weight"][i])
        nets.append(dict(net=net, required=cols["required"][i], level=cols["level"][i],
                         flatten_ok=bool(cols["flatten_ok"][i][0]), x=cols["x"][i], op=cols["op"][i],
                         dropped=int(cols["dropped"][i][0])))
    return nets


@pytest.fixture(scope="session")
def verify_corpus():
    """The reference `verify` recipe corpus with its golden op arrays."""
    import paper_2005_04347_b200 as A
    d = load_golden("verify_corpus.npz")
    xs = split(d["x"], d["x_len"])
    ops = split(d["op"], d["op_len"])
    mems = split(d["members"], d["members_len"])
    out = []
    for i, row in enumerate(d["spec"]):
        spec = A.GenSpec(int(row[0]), int(row[1]), int(row[2]), int(row[3]), int(row[4]), -1.0, 1.0,
                         int(row[5]))
        sizes = [int(s) for s in d["layer_sizes"][i] if s]
        out.append(dict(spec=spec, x=xs[i], op=ops[i], members=mems[i], layer_sizes=sizes,
                        csr_digest=str(d["csr_digest"][i])))
    return out


def bitwise_equal(a: np.ndarray, b: np.ndarray) -> bool:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def rel_close(g: np.ndarray, r: np.ndarray, rtol: float = 1e-5) -> np.ndarray:
    """SURVEY.md 8c parity rule: |g-r| <= rtol*|r|, or |r| < FLT_MIN and
    |g-r| <= rtol (denormal clamp values)."""
    g = g.astype(np.float64)
    r = r.astype(np.float64)
    d = np.abs(g - r)
    tiny = np.abs(r) < np.finfo(np.float32).tiny
    return np.where(tiny, d <= rtol, d <= rtol * np.abs(r))
