"""oracle/bind.py -- TEST INFRASTRUCTURE ONLY.

ctypes access to the two CPU checkers:
  * Oracle: oracle/liboracle.so, the plain-C restatement (asnn_oracle.c);
  * Ref:    oracle/_ref/libasnn_ref.so, the unmodified reference compiled from
            /root/reference by oracle/Makefile (present here and on the GPU box
            when build() ran with the reference checkout available).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libasnn_ref.so"

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
UNASSIGNED = 0xFFFFFFFF


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


def build_oracle():
    """Compile oracle/liboracle.so (and _ref when the reference is present)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


class Oracle:
    """The C restatement (asnn_oracle.c)."""

    def __init__(self):
        if not ORACLE_SO.exists():
            build_oracle()
        L = C.CDLL(str(ORACLE_SO))
        L.orc_sigmoid32.restype = C.c_float
        L.orc_sigmoid32.argtypes = [C.c_float]
        L.orc_sigmoid32_many.argtypes = [f32p, f32p, C.c_uint64]
        L.orc_compute_required.restype = C.c_int
        L.orc_compute_required.argtypes = [C.c_uint32, u32p, C.c_uint32, u32p, C.c_uint64, u32p,
                                           u32p, u8p]
        L.orc_segment.restype = C.c_int64
        L.orc_segment.argtypes = [C.c_uint32, u32p, C.c_uint32, u32p, C.c_uint64, u32p, u32p, u8p,
                                  u32p]
        L.orc_flatten.restype = C.c_int
        L.orc_flatten.argtypes = [C.c_uint32, u32p, C.c_uint32, u32p, C.c_uint64, u32p, u32p, f32p,
                                  u32p, C.c_uint32, u32p, u32p, u64p, u32p, f32p, u32p, u64p, u32p]
        L.orc_eval_sequential_batch.restype = C.c_int
        L.orc_eval_sequential_batch.argtypes = [C.c_uint32, u32p, C.c_uint32, u64p, u32p, f32p,
                                                C.c_uint32, u32p, C.c_uint32, f32p, C.c_uint32,
                                                C.c_uint32, f32p]
        L.orc_recompute.restype = None
        L.orc_recompute.argtypes = [C.c_uint32, u32p, u64p, u32p, f32p, u32p, C.c_uint32, f32p,
                                    f32p, u32p, C.c_uint64, f32p]
        self.L = L

    def recompute(self, lay, x, op, positions):
        """Recompute the given flat positions from a finished op array."""
        positions = np.ascontiguousarray(positions, dtype=np.uint32)
        x = np.ascontiguousarray(x, dtype=np.float32)
        op = np.ascontiguousarray(op, dtype=np.float32)
        io = np.ascontiguousarray(lay["input_order"], dtype=np.uint32)
        out = np.zeros(len(positions), np.float32)
        self.L.orc_recompute(int(lay["layer_offsets"][1]), _p(lay["node_ids"], C.c_uint32),
                             _p(lay["row_ptr"], C.c_uint64), _p(lay["in_nodes"], C.c_uint32),
                             _p(lay["in_weights"], C.c_float), _p(io, C.c_uint32), len(io),
                             _p(x, C.c_float), _p(op, C.c_float), _p(positions, C.c_uint32),
                             len(positions), _p(out, C.c_float))
        return out

    def sigmoid32(self, x):
        scalar = np.ndim(x) == 0
        x = np.ascontiguousarray(np.atleast_1d(x), dtype=np.float32)
        out = np.empty_like(x)
        self.L.orc_sigmoid32_many(_p(x, C.c_float), _p(out, C.c_float), x.size)
        return out[0] if scalar else out

    def compute_required(self, net) -> np.ndarray:
        mask = np.zeros(len(net.nodes), np.uint8)
        rc = self.L.orc_compute_required(len(net.nodes), _p(net.nodes, C.c_uint32), len(net.outputs),
                                         _p(net.outputs, C.c_uint32), len(net.source),
                                         _p(net.source, C.c_uint32), _p(net.target, C.c_uint32),
                                         _p(mask, C.c_uint8))
        assert rc == 0
        return mask

    def segment(self, net, mask=None):
        if mask is None:
            mask = self.compute_required(net)
        level = np.zeros(len(net.nodes), np.uint32)
        n = self.L.orc_segment(len(net.nodes), _p(net.nodes, C.c_uint32), len(net.inputs),
                               _p(net.inputs, C.c_uint32), len(net.source),
                               _p(net.source, C.c_uint32), _p(net.target, C.c_uint32),
                               _p(mask, C.c_uint8), _p(level, C.c_uint32))
        assert n >= 1
        return level, int(n)

    def flatten(self, net, level, n_layers):
        """Returns a dict mirroring LayeredLayout, or raises ValueError('unassigned output')."""
        N, E = len(net.nodes), len(net.source)
        lo = np.zeros(n_layers + 1, np.uint32)
        ids = np.zeros(N, np.uint32)
        rp = np.zeros(N + 1, np.uint64)
        src = np.zeros(E, np.uint32)
        w = np.zeros(E, np.float32)
        na, drop, idb = C.c_uint32(), C.c_uint64(), C.c_uint32()
        rc = self.L.orc_flatten(N, _p(net.nodes, C.c_uint32), len(net.outputs),
                                _p(net.outputs, C.c_uint32), E, _p(net.source, C.c_uint32),
                                _p(net.target, C.c_uint32), _p(net.weight, C.c_float),
                                _p(level, C.c_uint32), n_layers, _p(lo, C.c_uint32),
                                _p(ids, C.c_uint32), _p(rp, C.c_uint64), _p(src, C.c_uint32),
                                _p(w, C.c_float), C.byref(na), C.byref(drop), C.byref(idb))
        if rc == 3:
            raise ValueError("unassigned output")
        assert rc == 0
        n = na.value
        e = int(rp[n])
        return dict(total_layers=n_layers, layer_offsets=lo, node_ids=ids[:n], row_ptr=rp[:n + 1],
                    in_nodes=src[:e], in_weights=w[:e], input_order=net.inputs.copy(),
                    dropped_connections=drop.value, id_bound=idb.value)

    def layout(self, net):
        level, n = self.segment(net)
        return self.flatten(net, level, n)

    def eval_batch(self, lay, X) -> np.ndarray:
        """eval_sequential for every row of X; returns OP [n_vec][id_bound]."""
        X = np.ascontiguousarray(X, dtype=np.float32)
        if X.ndim == 1:
            X = X[None, :]
        n_vec = X.shape[0]
        op = np.zeros((n_vec, lay["id_bound"]), np.float32)
        io = np.ascontiguousarray(lay["input_order"], dtype=np.uint32)
        rc = self.L.orc_eval_sequential_batch(
            len(lay["node_ids"]), _p(lay["node_ids"], C.c_uint32), int(lay["layer_offsets"][1]),
            _p(lay["row_ptr"], C.c_uint64), _p(lay["in_nodes"], C.c_uint32),
            _p(lay["in_weights"], C.c_float), len(io), _p(io, C.c_uint32), lay["id_bound"],
            _p(X, C.c_float), X.shape[1], n_vec, _p(op, C.c_float))
        if rc == 2:
            raise ValueError("arity")
        assert rc == 0
        return op


class Ref:
    """The unmodified reference (oracle/_ref/libasnn_ref.so)."""

    def __init__(self, path=None):
        so = pathlib.Path(path) if path else REF_SO
        if not so.exists():
            raise FileNotFoundError(f"{so} not built (needs /root/reference at build time)")
        L = C.CDLL(str(so))
        vp = C.c_void_p
        sig = {
            "ref_generate": (vp, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                  C.c_float, C.c_float, C.c_uint64, C.POINTER(C.c_int)]),
            "ref_max_connections": (C.c_uint64, [C.c_uint32] * 4),
            "ref_network": (vp, [C.c_uint32, u32p, C.c_uint32, u32p, C.c_uint32, u32p, C.c_uint64,
                                 u32p, u32p, f32p]),
            "ref_free": (None, [vp]),
            "ref_net_n_nodes": (C.c_uint32, [vp]),
            "ref_net_n_inputs": (C.c_uint32, [vp]),
            "ref_net_n_outputs": (C.c_uint32, [vp]),
            "ref_net_n_edges": (C.c_uint64, [vp]),
            "ref_net_copy": (None, [vp, u32p, u32p, u32p, u32p, u32p, f32p]),
            "ref_validate": (C.c_uint32, [vp]),
            "ref_preprocess": (C.c_int, [vp]),
            "ref_preprocess_timed": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                               C.POINTER(C.c_double)]),
            "ref_required_count": (C.c_uint32, [vp]),
            "ref_required_copy": (None, [vp, u32p]),
            "ref_n_layers": (C.c_uint32, [vp]),
            "ref_assigned_count": (C.c_uint32, [vp]),
            "ref_unassigned_count": (C.c_uint32, [vp]),
            "ref_assignment_copy": (None, [vp, u32p, u32p, u32p]),
            "ref_layout_node_count": (C.c_uint32, [vp]),
            "ref_layout_edge_count": (C.c_uint64, [vp]),
            "ref_layout_total_layers": (C.c_uint32, [vp]),
            "ref_layout_id_bound": (C.c_uint32, [vp]),
            "ref_layout_dropped": (C.c_uint64, [vp]),
            "ref_layout_copy": (None, [vp, u32p, u32p, u32p, u8p, u64p, u32p, f32p, u32p]),
            "ref_layout_from_csr": (vp, [C.c_uint32, u32p, C.c_uint32, u32p, u64p, u32p, f32p,
                                         C.c_uint32, u32p, C.c_uint32]),
            "ref_eval_sequential": (C.c_int, [vp, f32p, C.c_uint32, f32p, f32p]),
            "ref_eval_parallel": (C.c_int, [vp, f32p, C.c_uint32, C.c_uint32, C.c_int, f32p]),
            "ref_eval_batch": (C.c_double, [vp, f32p, C.c_uint32, C.c_int, C.c_uint32, u32p,
                                            C.c_uint32, f32p]),
            "ref_max_threads": (C.c_int, []),
            "ref_layout_ptr": (vp, [vp]),
            "ref_sigmoid32_many": (None, [f32p, f32p, C.c_uint64]),
            "ref_parse": (vp, [C.c_char_p, C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int),
                               C.c_char_p, C.c_uint64]),
            "ref_serialize": (C.c_uint64, [vp, C.c_char_p, C.c_uint64]),
            "ref_from_chars_f32": (None, [C.c_char_p, u64p, C.c_uint64, f32p, u8p]),
            "ref_format_double": (None, [C.c_double, C.c_char_p, C.c_uint64]),
            "ref_validate_report": (C.c_uint32, [vp, C.c_char_p, C.c_uint64]),
            "ref_normalize": (vp, [vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        self.L = L

    # text format (io.cpp) ------------------------------------------------------
    def parse(self, text: bytes):
        """parse_network: (RefNet, None) or (None, (kind, line, message)),
        kind 1 = ParseError, 2 = ValidationError, 3 = other."""
        kind, line = C.c_int(0), C.c_int(0)
        err = C.create_string_buffer(1 << 16)
        h = self.L.ref_parse(text, len(text), C.byref(kind), C.byref(line), err, len(err))
        if h:
            return RefNet(self, h), None
        return None, (kind.value, line.value, err.value.decode())

    def serialize(self, rn: "RefNet") -> bytes:
        n = self.L.ref_serialize(rn.h, None, 0)
        if n == 0xFFFFFFFFFFFFFFFF:
            raise ValueError("serialize_network threw (invalid network)")
        buf = C.create_string_buffer(n)
        self.L.ref_serialize(rn.h, buf, n)
        return buf.raw[:n]

    def from_chars_f32(self, tokens):
        """std::from_chars<float> on each token: (values, status 0 ok / 1 error)."""
        enc = [t.encode() if isinstance(t, str) else t for t in tokens]
        off = np.zeros(len(enc) + 1, np.uint64)
        off[1:] = np.cumsum([len(t) for t in enc])
        buf = b"".join(enc)
        out = np.zeros(len(enc), np.float32)
        st = np.zeros(len(enc), np.uint8)
        self.L.ref_from_chars_f32(buf, _p(off, C.c_uint64), len(enc), _p(out, C.c_float),
                                  _p(st, C.c_uint8))
        return out, st

    def format_double(self, v: float) -> str:
        buf = C.create_string_buffer(64)
        self.L.ref_format_double(float(v), buf, 64)
        return buf.value.decode()

    # networks ---------------------------------------------------------------
    def generate(self, spec):
        err = C.c_int(0)
        h = self.L.ref_generate(spec.input_count, spec.output_count, spec.hidden_count,
                                spec.connection_count, spec.target_depth, spec.weight_min,
                                spec.weight_max, spec.seed & 0xFFFFFFFFFFFFFFFF, C.byref(err))
        if not h:
            raise ValueError(f"infeasible (code {err.value})")
        return RefNet(self, h)

    def network(self, net):
        h = self.L.ref_network(len(net.nodes), _p(net.nodes, C.c_uint32), len(net.inputs),
                               _p(net.inputs, C.c_uint32), len(net.outputs),
                               _p(net.outputs, C.c_uint32), len(net.source),
                               _p(net.source, C.c_uint32), _p(net.target, C.c_uint32),
                               _p(net.weight, C.c_float))
        return RefNet(self, h)

    def layout_from_csr(self, lay):
        io = np.ascontiguousarray(lay["input_order"], dtype=np.uint32)
        h = self.L.ref_layout_from_csr(lay["total_layers"], _p(lay["layer_offsets"], C.c_uint32),
                                       len(lay["node_ids"]), _p(lay["node_ids"], C.c_uint32),
                                       _p(lay["row_ptr"], C.c_uint64),
                                       _p(lay["in_nodes"], C.c_uint32),
                                       _p(lay["in_weights"], C.c_float), len(io),
                                       _p(io, C.c_uint32), lay["id_bound"])
        return RefNet(self, h)

    def sigmoid32(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty_like(x)
        self.L.ref_sigmoid32_many(_p(x, C.c_float), _p(out, C.c_float), x.size)
        return out


class RefNet:
    def __init__(self, ref: Ref, h):
        self.ref, self.L, self.h = ref, ref.L, h

    def __del__(self):
        try:
            self.L.ref_free(self.h)
        except Exception:
            pass

    def arrays(self):
        L, h = self.L, self.h
        n, i, o, e = L.ref_net_n_nodes(h), L.ref_net_n_inputs(h), L.ref_net_n_outputs(h), L.ref_net_n_edges(h)
        nodes, ins, outs = np.zeros(n, np.uint32), np.zeros(i, np.uint32), np.zeros(o, np.uint32)
        src, dst, w = np.zeros(e, np.uint32), np.zeros(e, np.uint32), np.zeros(e, np.float32)
        L.ref_net_copy(h, _p(nodes, C.c_uint32), _p(ins, C.c_uint32), _p(outs, C.c_uint32),
                       _p(src, C.c_uint32), _p(dst, C.c_uint32), _p(w, C.c_float))
        return dict(nodes=nodes, inputs=ins, outputs=outs, source=src, target=dst, weight=w)

    def validate_report(self) -> list:
        buf = C.create_string_buffer(1 << 20)
        n = self.L.ref_validate_report(self.h, buf, len(buf))
        return buf.value.decode().split("\n") if n else []

    def normalize(self) -> "RefNet":
        return RefNet(self.ref, self.L.ref_normalize(self.h))

    def validate(self) -> int:
        return self.L.ref_validate(self.h)

    def preprocess(self) -> int:
        return self.L.ref_preprocess(self.h)

    def preprocess_timed(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        rc = self.L.ref_preprocess_timed(self.h, C.byref(a), C.byref(b), C.byref(c))
        return rc, (a.value, b.value, c.value)

    def required(self) -> np.ndarray:
        m = np.zeros(self.L.ref_required_count(self.h), np.uint32)
        self.L.ref_required_copy(self.h, _p(m, C.c_uint32))
        return m

    def assignment(self):
        nl = self.L.ref_n_layers(self.h)
        sizes = np.zeros(nl, np.uint32)
        members = np.zeros(self.L.ref_assigned_count(self.h), np.uint32)
        un = np.zeros(self.L.ref_unassigned_count(self.h), np.uint32)
        self.L.ref_assignment_copy(self.h, _p(sizes, C.c_uint32), _p(members, C.c_uint32),
                                   _p(un, C.c_uint32))
        bounds = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        return [members[bounds[k]:bounds[k + 1]] for k in range(nl)], un

    def layout(self):
        L, h = self.L, self.h
        n, e, tl = L.ref_layout_node_count(h), L.ref_layout_edge_count(h), L.ref_layout_total_layers(h)
        lo = np.zeros(tl + 1, np.uint32)
        ids, lay, sens = np.zeros(n, np.uint32), np.zeros(n, np.uint32), np.zeros(n, np.uint8)
        rp = np.zeros(n + 1, np.uint64)
        src, w = np.zeros(e, np.uint32), np.zeros(e, np.float32)
        io = np.zeros(L.ref_net_n_inputs(h), np.uint32)
        L.ref_layout_copy(h, _p(lo, C.c_uint32), _p(ids, C.c_uint32), _p(lay, C.c_uint32),
                          _p(sens, C.c_uint8), _p(rp, C.c_uint64), _p(src, C.c_uint32),
                          _p(w, C.c_float), _p(io, C.c_uint32))
        return dict(total_layers=tl, layer_offsets=lo, node_ids=ids, node_layer=lay, is_sensor=sens,
                    row_ptr=rp, in_nodes=src, in_weights=w, input_order=io,
                    dropped_connections=L.ref_layout_dropped(h), id_bound=L.ref_layout_id_bound(h))

    def eval_sequential(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        idb = self.L.ref_layout_id_bound(self.h)
        si, so = np.zeros(idb, np.float32), np.zeros(idb, np.float32)
        rc = self.L.ref_eval_sequential(self.h, _p(x, C.c_float), len(x), _p(si, C.c_float),
                                        _p(so, C.c_float))
        if rc:
            raise ValueError(f"ref eval failed ({rc})")
        return si, so

    def eval_parallel(self, x, workers=0, backend=0):
        x = np.ascontiguousarray(x, dtype=np.float32)
        so = np.zeros(self.L.ref_layout_id_bound(self.h), np.float32)
        rc = self.L.ref_eval_parallel(self.h, _p(x, C.c_float), len(x), workers, backend,
                                      _p(so, C.c_float))
        return rc, so

    def eval_batch(self, X, mode: int, workers: int = 0, out_ids=None):
        """Seconds for the batch (mode 0 seq / 1 eval_parallel / 2 omp loop)."""
        X = np.ascontiguousarray(X, dtype=np.float32)
        out = None
        if out_ids is not None:
            out_ids = np.ascontiguousarray(out_ids, dtype=np.uint32)
            out = np.zeros((X.shape[0], len(out_ids)), np.float32)
        t = self.L.ref_eval_batch(self.h, _p(X, C.c_float), X.shape[0], mode, workers,
                                  _p(out_ids, C.c_uint32), 0 if out_ids is None else len(out_ids),
                                  _p(out, C.c_float))
        if t < 0:
            raise ValueError(f"ref eval failed ({-t})")
        return t, out


def available_ref() -> bool:
    return REF_SO.exists()


REF_DEV_SO = HERE / "_ref" / "libasnn_ref_dev.so"


class RefDev(Ref):
    """The reference plus the maintainer's DeviceCompute binding
    (integration/asnn_device_backend.cpp) linked against libasnn_b200.so."""

    def __init__(self):
        super().__init__(REF_DEV_SO)
        self.L.ref_dev_eval.restype = C.c_int
        self.L.ref_dev_eval.argtypes = [C.c_void_p, f32p, C.c_uint32, f32p]

    def timed(self, rn: "RefNet", x, resident: bool, warmup: int, reps: int):
        """(mean_us, stddev_us) of eval_parallel(DeviceCompute) per call
        (resident=False) or of asnn_dev_activate on a layout uploaded once
        (resident=True), timed inside C++ (integration/asnn_device_backend.cpp)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        m, sd = C.c_double(), C.c_double()
        fn = self.L.ref_dev_resident_timed if resident else self.L.ref_dev_eval_timed
        fn.restype = C.c_int
        fn.argtypes = [C.c_void_p, f32p, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_double),
                       C.POINTER(C.c_double)]
        rc = fn(self.L.ref_layout_ptr(rn.h), _p(x, C.c_float), len(x), warmup, reps, C.byref(m), C.byref(sd))
        if rc:
            raise RuntimeError(f"device timing failed ({rc})")
        return m.value, sd.value

    def server_timed(self, rn: "RefNet", x, warmup: int, reps: int):
        """(mean_us, stddev_us) of one vector through the resident server
        (asnn_dev_server_activate, declared outputs back), timed inside C++;
        None when the network does not fit one SM's shared memory."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        outs = np.ascontiguousarray(rn.arrays()["outputs"], dtype=np.uint32)
        m, sd = C.c_double(), C.c_double()
        fn = self.L.ref_dev_server_timed
        fn.restype = C.c_int
        fn.argtypes = [C.c_void_p, u32p, C.c_uint32, f32p, C.c_uint32, C.c_uint32, C.c_uint32,
                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
        rc = fn(self.L.ref_layout_ptr(rn.h), _p(outs, C.c_uint32), len(outs), _p(x, C.c_float), len(x), warmup,
                reps, C.byref(m), C.byref(sd))
        if rc == 1:
            return None
        if rc:
            raise RuntimeError(f"server timing failed ({rc})")
        return m.value, sd.value

    def eval_device(self, rn: "RefNet", x):
        """eval_parallel(..., DeviceCompute) on the reference's own LayeredLayout."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.zeros(self.L.ref_layout_id_bound(rn.h), np.float32)
        rc = self.L.ref_dev_eval(self.L.ref_layout_ptr(rn.h), _p(x, C.c_float), len(x),
                                 _p(out, C.c_float))
        return rc, out


def available_ref_dev() -> bool:
    return REF_DEV_SO.exists()


# --- bench corpora for the CPU legs (oracle/libcorpus.so) ------------------------------
CORPUS_SO = HERE / "libcorpus.so"


class SplitMix64:
    """rng.hpp:10-38 (seeds of the config-5 population, like the reference)."""
    M = 0xFFFFFFFFFFFFFFFF

    def __init__(self, seed: int):
        self.s = seed & self.M

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & self.M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)


class NetArrays:
    """A network as plain arrays (network.hpp:12-32 fields)."""

    def __init__(self, nodes, inputs, outputs, source, target, weight):
        self.nodes, self.inputs, self.outputs = nodes, inputs, outputs
        self.source, self.target, self.weight = source, target, weight


class _NetDesc(C.Structure):
    _fields_ = [("n_nodes", C.c_uint32), ("nodes", u32p), ("n_inputs", C.c_uint32),
                ("inputs", u32p), ("n_outputs", C.c_uint32), ("outputs", u32p),
                ("n_connections", C.c_uint64), ("source", u32p), ("target", u32p),
                ("weight", f32p)]


class Corpus:
    """The bench's seeded generators compiled from csrc/netgen.cpp into
    oracle/libcorpus.so (no device code, no engine): configs 2 and 4."""

    def __init__(self):
        if not CORPUS_SO.exists():
            raise FileNotFoundError(f"{CORPUS_SO} not built (make -C oracle)")
        L = C.CDLL(str(CORPUS_SO))
        vp = C.c_void_p
        L.asnn_gen_mlp.restype = C.c_int
        L.asnn_gen_mlp.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64, C.POINTER(vp)]
        L.asnn_gen_powerlaw.restype = C.c_int
        L.asnn_gen_powerlaw.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                        C.c_double, C.c_uint64, C.POINTER(vp)]
        L.asnn_corpus_desc.restype = C.c_int
        L.asnn_corpus_desc.argtypes = [vp, C.POINTER(_NetDesc)]
        L.asnn_corpus_free.restype = None
        L.asnn_corpus_free.argtypes = [vp]
        self.L = L

    def _take(self, h) -> NetArrays:
        d = _NetDesc()
        self.L.asnn_corpus_desc(h, C.byref(d))

        def arr(p, n, dt):
            return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, dt)
        net = NetArrays(arr(d.nodes, d.n_nodes, np.uint32), arr(d.inputs, d.n_inputs, np.uint32),
                        arr(d.outputs, d.n_outputs, np.uint32),
                        arr(d.source, d.n_connections, np.uint32),
                        arr(d.target, d.n_connections, np.uint32),
                        arr(d.weight, d.n_connections, np.float32))
        self.L.asnn_corpus_free(h)
        return net

    def mlp(self, layers, width, p, seed) -> NetArrays:
        h = C.c_void_p()
        assert self.L.asnn_gen_mlp(layers, width, p, seed, C.byref(h)) == 0
        return self._take(h)

    def powerlaw(self, n_nodes, bands, n_in, n_out, target_edges, alpha, seed) -> NetArrays:
        h = C.c_void_p()
        assert self.L.asnn_gen_powerlaw(n_nodes, bands, n_in, n_out, target_edges, alpha, seed,
                                        C.byref(h)) == 0
        return self._take(h)
