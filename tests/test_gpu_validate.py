"""validate / normalize of in-memory networks on the device
(asnn_dev_validate / asnn_dev_normalize, csrc/parse.cu) against the
reference's own functions (network.cpp:69-85, 151-216, oracle/_ref): the same
violation messages in the same order, the same remapped network."""
from __future__ import annotations

import random

import numpy as np
import pytest

import paper_2005_04347_b200 as A

pytestmark = pytest.mark.gpu


def net(nodes, inputs, outputs, conns):
    src = [c[0] for c in conns]
    dst = [c[1] for c in conns]
    w = [c[2] if len(c) > 2 else 0.5 for c in conns]
    return A.Network(np.asarray(nodes, np.uint32), inputs, outputs, src, dst, w)


CASES = [
    net([0, 1, 2], [0], [2], [(0, 1), (1, 2)]),                                     # valid
    net([0, 1, 2], [], [2], [(0, 1), (1, 2)]),                                      # empty inputs
    net([0, 1, 2], [0], [], [(0, 1), (1, 2)]),                                      # empty outputs
    net([0, 1, 2, 3], [0, 1, 0, 9, 0], [2, 2, 7], [(0, 2), (1, 2)]),                # dup / unknown declarations
    net([0, 1, 2, 3], [0, 1], [1, 3, 0], [(0, 3), (1, 3)]),                         # overlap
    net([0, 1, 2], [0], [2], [(0, 5), (7, 2), (1, 1), (0, 1), (0, 1), (1, 2), (2, 0), (0, 1)]),
    net([0, 1, 2, 3, 4], [0], [4], [(0, 1), (1, 2), (2, 3), (3, 1), (3, 4)]),        # cycle
    net([0, 1, 2, 3, 4, 5, 6], [0], [6], [(0, 6), (4, 5), (5, 4), (2, 3), (3, 2)]),   # first cycle by DFS order
    net([0, 1, 2], [0, 1], [2], [(0, 2), (2, 1), (1, 2), (2, 2), (3, 4)]),           # everything at once
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_validate_cases(ref, i):
    n = CASES[i]
    assert A.validate(n) == ref.network(n).validate_report()


def test_validate_random_damage(ref):
    rng = random.Random(11)
    for trial in range(40):
        base = A.generate(A.random_spec(A.SplitMix64(trial), 200, 3000))
        src, dst = list(base.source), list(base.target)
        nodes, ins, outs = list(base.nodes), list(base.inputs), list(base.outputs)
        for _ in range(rng.randint(0, 6)):
            op = rng.randrange(6)
            k = rng.randrange(len(src))
            if op == 0:
                src.insert(k, src[k]); dst.insert(k, dst[k])           # duplicate connection
            elif op == 1:
                src.append(dst[k]); dst.append(src[k])                  # back edge: cycle
            elif op == 2:
                src.append(src[k]); dst.append(src[k])                  # self-loop
            elif op == 3:
                src.append(max(nodes) + 5); dst.append(dst[k])          # unknown node
            elif op == 4:
                src.append(src[k]); dst.append(ins[0])                  # input with incoming
            else:
                outs.append(ins[-1])                                    # overlap
        n = A.Network(np.asarray(nodes, np.uint32), ins, outs, src, dst, np.full(len(src), 0.25, np.float32))
        assert A.validate(n) == ref.network(n).validate_report(), trial


def test_normalize_matches_reference(ref):
    for seed in range(5):
        n0 = A.generate(A.random_spec(A.SplitMix64(50 + seed), 100, 2000))
        shift = np.uint32(1000 * (seed + 1))
        n = A.Network(n0.nodes * 3 + shift, n0.inputs * 3 + shift, n0.outputs * 3 + shift,
                      n0.source * 3 + shift, n0.target * 3 + shift, n0.weight)
        got = A.normalize(n)
        want = ref.network(n).normalize().arrays()
        for k in ("nodes", "inputs", "outputs", "source", "target"):
            assert np.array_equal(getattr(got, k), want[k]), k
        assert np.array_equal(got.weight.view(np.uint32), want["weight"].view(np.uint32))
