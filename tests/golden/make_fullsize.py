"""Full-size golden fixtures from the UNMODIFIED reference (TEST INFRASTRUCTURE).

Run here, where /root/reference is present (needs ~30 GB of RAM and ~25 min of
one CPU core for config 4's preprocessing):

    make -C oracle && python tests/golden/make_fullsize.py [c1] [c4]

For each config the network is the bench corpus (`bench.make_network`, seeded);
the reference's own compute_required / segment / flatten (network.cpp:222-255,
segmentation.cpp:20-101, layout.cpp:12-83) run on it through oracle/_ref, and
its eval_parallel (eval.cpp:49-80, all host threads; par == seq bitwise is
pinned by test_eval.cpp:136-149) evaluates every vector of the config's batch.
Written to tests/golden/fullsize_<cfg>.npz (small: digests + declared outputs):

  layout_sha256     sha256 over layer_offsets(u32) | node_ids(u32) | row_ptr(u64)
                    | in_nodes(u32) | in_weights(u32 bits) | input_order(u32)
  dropped, id_bound, total_layers, node_count, edge_count
  required_count    |compute_required(net).members|
  x                 the batch ([B][n_in] f32, np.random.default_rng(seed))
  state_sha256      per vector: sha256 of the id-indexed op array (id_bound f32)
  outputs           [B][n_out] read_outputs (bitwise reference values)
  ref_preprocess_s  the reference's own preprocessing times (required, segment,
                    flatten), for DESIGN.md's comparison

tests/test_gpu_fullsize.py compares the device layout and every vector's full
state with these bit for bit (no /root/reference on the GPU box).
"""
from __future__ import annotations

import hashlib
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

OUT = pathlib.Path(__file__).resolve().parent

# cfg -> (batch, input seed); the GPU test draws the same batch
BATCH = {"c1": (64, 1), "c4": (64, 4)}


def layout_digest(lay: dict) -> str:
    h = hashlib.sha256()
    for k, dt in (("layer_offsets", np.uint32), ("node_ids", np.uint32), ("row_ptr", np.uint64),
                  ("in_nodes", np.uint32)):
        h.update(np.ascontiguousarray(lay[k], dtype=dt).tobytes())
    h.update(np.ascontiguousarray(lay["in_weights"], dtype=np.float32).view(np.uint32).tobytes())
    h.update(np.ascontiguousarray(lay["input_order"], dtype=np.uint32).tobytes())
    return h.hexdigest()


def state_digest(op: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(op, dtype=np.float32).view(np.uint32).tobytes()).hexdigest()


def batch_inputs(cfg: str, n_in: int) -> np.ndarray:
    B, seed = BATCH[cfg]
    return np.random.default_rng(seed).uniform(-2, 2, (B, n_in)).astype(np.float32)


def make(cfg: str):
    import bench
    from oracle.bind import Ref
    ref = Ref()
    t0 = time.perf_counter()
    net = bench.make_network(cfg, 1.0)[0]
    print(f"[{cfg}] generated {len(net.source)} edges in {time.perf_counter() - t0:.1f}s", flush=True)
    outputs = np.array(net.outputs, np.uint32)
    n_in = len(net.inputs)
    rn = ref.network(net)
    del net
    t0 = time.perf_counter()
    rc, (t_req, t_seg, t_flat) = rn.preprocess_timed()
    assert rc == 0, rc
    print(f"[{cfg}] reference preprocessing {time.perf_counter() - t0:.1f}s "
          f"(required {t_req:.1f} segment {t_seg:.1f} flatten {t_flat:.1f})", flush=True)
    required_count = len(rn.required())
    lay = rn.layout()
    dig = layout_digest(lay)
    X = batch_inputs(cfg, n_in)
    states, outs = [], []
    t0 = time.perf_counter()
    for b in range(X.shape[0]):
        rc, op = rn.eval_parallel(X[b])
        assert rc == 0, rc
        states.append(state_digest(op))
        outs.append(op[outputs])
    print(f"[{cfg}] {X.shape[0]} vectors by eval_parallel in {time.perf_counter() - t0:.1f}s", flush=True)
    np.savez_compressed(
        OUT / f"fullsize_{cfg}.npz", layout_sha256=np.array(dig),
        dropped=np.uint64(lay["dropped_connections"]), id_bound=np.uint32(lay["id_bound"]),
        total_layers=np.uint32(lay["total_layers"]), node_count=np.uint32(len(lay["node_ids"])),
        edge_count=np.uint64(len(lay["in_nodes"])), required_count=np.uint32(required_count),
        x=X, state_sha256=np.array(states), outputs=np.stack(outs),
        ref_preprocess_s=np.array([t_req, t_seg, t_flat]))
    print(f"[{cfg}] layout {dig}", flush=True)


if __name__ == "__main__":
    for c in (sys.argv[1:] or list(BATCH)):
        make(c)
