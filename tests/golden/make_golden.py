"""Generates tests/golden/*.npz from the UNMODIFIED reference.

Run here (the reference checkout must be present):
    make -C oracle && python tests/golden/make_golden.py

Fixtures written:
  verify_corpus.npz  -- the reference `asnn verify` recipe (asnn_main.cpp:233-297,
                        seed 20260810 like acceptance.cpp:74-75, 100..20000
                        connections): per trial the GenSpec, the input vector,
                        segment() levels (as layer sizes + members), flatten()'s
                        CSR digest and eval_sequential's op array (bitwise);
  adversarial.npz    -- random DAGs with sparse ids, dead ends, source-less
                        hidden nodes and unreachable outputs:
                        the network arrays plus the reference's required set,
                        layers, unassigned list and (when flatten succeeds) op;
  sigmoid.npz        -- sigmoid32 of the reference on edge-case and random floats;
  corpus_digest.npz  -- sha256 of generate() output for a few specs.
"""
from __future__ import annotations

import hashlib
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.bind import Ref  # noqa: E402
import paper_2005_04347_b200 as A  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def verify_corpus(ref: Ref, trials=40, min_conn=100, max_conn=20000, seed=20260810):
    master = A.SplitMix64(seed)
    rec = {k: [] for k in ("spec", "x", "layer_sizes", "members", "csr_digest", "op", "op_len",
                           "x_len", "members_len")}
    for t in range(trials):
        net_seed = master.next()
        rng = A.SplitMix64(net_seed)
        conn = min_conn + rng.bounded(max_conn - min_conn + 1)
        depth = 3 + rng.bounded(2) if conn < 64 else 3 + rng.bounded(38)
        n_in = 1 + rng.bounded(8)
        n_out = 1 + rng.bounded(4)
        spec = A.corpus_spec(conn, depth, n_in, n_out, net_seed)
        rn = ref.generate(spec)
        assert rn.preprocess() == 0
        layers, _ = rn.assignment()
        lay = rn.layout()
        x = np.array([rng.uniform(-2.0, 2.0) for _ in range(len(lay["input_order"]))], np.float32)
        _, op = rn.eval_sequential(x)
        rec["spec"].append([spec.input_count, spec.output_count, spec.hidden_count,
                            spec.connection_count, spec.target_depth, spec.seed])
        rec["x"].append(x)
        rec["x_len"].append(len(x))
        rec["layer_sizes"].append(np.array([len(l) for l in layers] + [0] * (64 - len(layers)), np.uint32))
        mem = np.concatenate(layers).astype(np.uint32)
        rec["members"].append(mem)
        rec["members_len"].append(len(mem))
        rec["csr_digest"].append(digest(lay["layer_offsets"], lay["node_ids"], lay["row_ptr"],
                                        lay["in_nodes"], lay["in_weights"].view(np.uint32)))
        rec["op"].append(op)
        rec["op_len"].append(len(op))
    np.savez_compressed(
        OUT / "verify_corpus.npz",
        spec=np.array(rec["spec"], np.uint64), x=np.concatenate(rec["x"]),
        x_len=np.array(rec["x_len"]), layer_sizes=np.stack(rec["layer_sizes"]),
        members=np.concatenate(rec["members"]), members_len=np.array(rec["members_len"]),
        csr_digest=np.array(rec["csr_digest"]), op=np.concatenate(rec["op"]),
        op_len=np.array(rec["op_len"]))


def adversarial_net(rng: np.random.Generator):
    """Random DAG over sparse ids: topological order = a random permutation."""
    n = int(rng.integers(5, 200))
    ids = np.sort(rng.choice(np.arange(0, 10 * n), size=n, replace=False)).astype(np.uint32)
    order = rng.permutation(n)
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    n_in = int(rng.integers(1, max(2, n // 5)))
    inputs = ids[order[:n_in]]
    m = int(rng.integers(n, 6 * n))
    a = rng.integers(0, n, size=m)
    b = rng.integers(0, n, size=m)
    keep = rank[a] < rank[b]
    a, b = a[keep], b[keep]
    pairs = np.unique(np.stack([a, b], 1), axis=0)
    # no edges into inputs (validate(): InputHasIncoming)
    in_set = set(inputs.tolist())
    pairs = np.array([p for p in pairs if int(ids[p[1]]) not in in_set], np.int64).reshape(-1, 2)
    if rng.random() < 0.6:
        # mostly evaluable: every non-input node not first in topological
        # order gets one predecessor earlier in that order (some remain
        # source-less when their only candidates are dead ends)
        has_in = set(pairs[:, 1].tolist())
        extra = []
        for r in range(1, n):
            v = order[r]
            if int(ids[v]) in in_set or v in has_in or rng.random() < 0.05:
                continue
            extra.append((order[int(rng.integers(0, r))], v))
        if extra:
            pairs = np.unique(np.concatenate([pairs, np.array(extra, np.int64)]), axis=0)
    rng.shuffle(pairs)
    src, dst = ids[pairs[:, 0]], ids[pairs[:, 1]]
    w = rng.uniform(-1.5, 1.5, size=len(src)).astype(np.float32)
    cand = np.setdiff1d(ids, inputs)
    n_out = int(rng.integers(1, min(5, len(cand)) + 1)) if len(cand) else 0
    outputs = rng.choice(cand, size=n_out, replace=False).astype(np.uint32) if n_out else \
        np.zeros(0, np.uint32)
    return A.Network(ids, inputs, outputs, src, dst, w)


def adversarial(ref: Ref, count=300, seed=7):
    rng = np.random.default_rng(seed)
    fields = {k: [] for k in ("nodes", "inputs", "outputs", "source", "target", "weight",
                              "required", "level", "flatten_ok", "x", "op", "dropped")}
    lens = {k: [] for k in fields}
    for _ in range(count):
        net = adversarial_net(rng)
        rn = ref.network(net)
        rc = rn.preprocess()
        req = rn.required()
        layers, _ = rn.assignment()
        level = np.full(len(net.nodes), 0xFFFFFFFF, np.uint32)
        for l, mem in enumerate(layers):
            level[np.searchsorted(net.nodes, mem)] = l
        x = rng.uniform(-2, 2, size=len(net.inputs)).astype(np.float32)
        if rc == 0:
            _, op = rn.eval_sequential(x)
            dropped = rn.layout()["dropped_connections"]
        else:
            op = np.zeros(0, np.float32)
            dropped = 0
        vals = dict(nodes=net.nodes, inputs=net.inputs, outputs=net.outputs, source=net.source,
                    target=net.target, weight=net.weight, required=req, level=level,
                    flatten_ok=np.array([rc == 0], np.uint8), x=x, op=op,
                    dropped=np.array([dropped], np.uint64))
        for k, v in vals.items():
            fields[k].append(np.asarray(v))
            lens[k].append(len(np.asarray(v)))
    np.savez_compressed(OUT / "adversarial.npz",
                        **{k: np.concatenate(v) for k, v in fields.items()},
                        **{k + "_len": np.array(v) for k, v in lens.items()})


def sigmoid(ref: Ref):
    rng = np.random.default_rng(11)
    special = np.array([0.0, -0.0, 0.5, 1.0, -1.0, 0.125, 0.4, 200.0, -200.0, 1e-30, -1e-30,
                        1.4e-45, -1.4e-45, 3.4e38, -3.4e38, np.inf, -np.inf, 7.5, -7.5, 8.0, -8.0,
                        15.0, -15.0, 20.0, -20.0, 150.0, -150.0], np.float32)
    rand = np.concatenate([rng.uniform(-25, 25, 40000), rng.normal(0, 2, 40000)]).astype(np.float32)
    bits = rng.integers(0, 2**32, size=40000, dtype=np.uint64).astype(np.uint32).view(np.float32)
    bits = bits[np.isfinite(bits)]
    x = np.concatenate([special, rand, bits])
    np.savez_compressed(OUT / "sigmoid.npz", x=x, y=ref.sigmoid32(x))


def corpus_digest(ref: Ref):
    specs = [A.GenSpec(16, 4, 980, 10000, 10, -1.0, 1.0, 1),
             A.GenSpec(3, 2, 0, 6, 2, -1.0, 1.0, 5),
             A.GenSpec(4, 2, 30, 500, 6, -1.0, 1.0, 9),        # dense branch
             A.GenSpec(8, 4, 188, 1000, 8, -1.0, 1.0, 0xDEADBEEF),
             A.GenSpec(16, 4, 4980, 50000, 200, -0.5, 0.25, 3)]
    rows, digs = [], []
    for s in specs:
        a = ref.generate(s).arrays()
        rows.append([s.input_count, s.output_count, s.hidden_count, s.connection_count,
                     s.target_depth, s.seed])
        digs.append(digest(a["nodes"], a["inputs"], a["outputs"], a["source"], a["target"],
                           a["weight"].view(np.uint32)))
    np.savez_compressed(OUT / "corpus_digest.npz", spec=np.array(rows, np.uint64),
                        wrange=np.array([[s.weight_min, s.weight_max] for s in specs], np.float32),
                        digest=np.array(digs))


if __name__ == "__main__":
    ref = Ref()
    verify_corpus(ref)
    adversarial(ref)
    sigmoid(ref)
    corpus_digest(ref)
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
