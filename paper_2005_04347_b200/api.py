"""Python mirror of the reference's hot-path API, backed by the sm_100a engine.

Names, argument meaning and error behaviour follow /root/reference/proj:

  make_network          network.cpp:39-55
  compute_required      network.cpp:222-255      -> asnn_dev_compute_required (GPU)
  segment               segmentation.cpp:20-101  -> asnn_dev_segment (GPU Kahn)
  flatten               layout.cpp:12-83         -> asnn_dev_flatten (GPU CSR build)
  eval_parallel         eval.cpp:49-80           -> Backend.DeviceCompute only:
                                                    asnn_dev_upload_layout + asnn_dev_activate
  read_outputs          eval.cpp:82-87
  layer_slice_bounds    layout.cpp:85-91
  max_layer_width       eval.cpp:89-94
  depth / unassigned_outputs / LayerAssignment.layer_of   segmentation.cpp:7-12,103-112
  generate              netgen.cpp:71-157        -> asnn_gen_reference (host corpus tool)

Exceptions mirror errors.hpp:9-55.  There is no host evaluator here: the
HostParallel backend and eval_sequential belong to the reference (the
oracle in tests/), and asking this package for them raises
BackendUnavailable instead of silently computing on the CPU.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import f32p, u8p, u32p, u64p


# --- errors.hpp:9-55 --------------------------------------------------------
class AsnnError(RuntimeError):
    pass


class InputArityMismatch(AsnnError):
    pass


class OutputUnreachable(AsnnError):
    pass


UnassignedOutput = OutputUnreachable


class LayerOutOfRange(IndexError):
    pass


class BackendUnavailable(AsnnError):
    pass


class InfeasibleSpec(AsnnError):
    pass


class DeviceError(AsnnError):
    pass


class IoError(AsnnError):
    pass


class ParseError(AsnnError):
    """errors.hpp:31-35: what() = "line N: ...", .line = N."""

    def __init__(self, msg: str, line: int = 0):
        super().__init__(msg)
        self.line = line


class ValidationError(AsnnError):
    """errors.hpp:37-53: what() = "invalid network\n  v1\n  v2 ...", .violations."""

    def __init__(self, msg: str):
        super().__init__(msg)
        self.violations = msg.split("\n  ")[1:]


def _raise(rc: int, msg: str):
    cls = {
        _lib.ASNN_E_UNAVAILABLE: BackendUnavailable,
        _lib.ASNN_E_ARITY: InputArityMismatch,
        _lib.ASNN_E_UNASSIGNED_OUTPUT: OutputUnreachable,
        _lib.ASNN_E_LAYER_RANGE: LayerOutOfRange,
        _lib.ASNN_E_INFEASIBLE: InfeasibleSpec,
        _lib.ASNN_E_INVALID: ValueError,
        _lib.ASNN_E_VALIDATION: ValidationError,
        _lib.ASNN_E_IO: IoError,
    }.get(rc, DeviceError)
    raise cls(msg or f"asnn status {rc}")


# --- data model: network.hpp:12-32 -----------------------------------------
def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32).reshape(-1))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1))


@dataclass
class Network:
    """Network (network.hpp:25-32) with SoA connections."""
    nodes: np.ndarray
    inputs: np.ndarray
    outputs: np.ndarray
    source: np.ndarray
    target: np.ndarray
    weight: np.ndarray

    def __post_init__(self):
        self.nodes = _u32(self.nodes)
        self.inputs = _u32(self.inputs)
        self.outputs = _u32(self.outputs)
        self.source = _u32(self.source)
        self.target = _u32(self.target)
        self.weight = _f32(self.weight)

    @property
    def connections(self):
        return list(zip(self.source.tolist(), self.target.tolist(), self.weight.tolist()))

    def desc(self) -> _lib.NetworkDesc:
        d = _lib.NetworkDesc()
        d.n_nodes = len(self.nodes)
        d.nodes = _lib.ptr(self.nodes, C.c_uint32)
        d.n_inputs = len(self.inputs)
        d.inputs = _lib.ptr(self.inputs, C.c_uint32)
        d.n_outputs = len(self.outputs)
        d.outputs = _lib.ptr(self.outputs, C.c_uint32)
        d.n_connections = len(self.source)
        d.source = _lib.ptr(self.source, C.c_uint32)
        d.target = _lib.ptr(self.target, C.c_uint32)
        d.weight = _lib.ptr(self.weight, C.c_float)
        return d


def make_network(inputs, outputs, connections, extra_nodes=()) -> Network:
    """network.cpp:39-55: node set = union of inputs, outputs, endpoints."""
    conns = list(connections)
    src = np.array([c[0] for c in conns], dtype=np.uint32)
    dst = np.array([c[1] for c in conns], dtype=np.uint32)
    w = np.array([c[2] for c in conns], dtype=np.float32)
    nodes = np.unique(np.concatenate([_u32(extra_nodes), _u32(inputs), _u32(outputs), src, dst]))
    return Network(nodes, inputs, outputs, src, dst, w)


@dataclass
class RequiredSet:
    """RequiredSet (network.hpp:100-104)."""
    members: np.ndarray

    def contains(self, node_id: int) -> bool:
        i = np.searchsorted(self.members, node_id)
        return bool(i < len(self.members) and self.members[i] == node_id)


@dataclass
class LayerAssignment:
    """LayerAssignment (segmentation.hpp:14-21)."""
    layers: list
    unassigned: np.ndarray
    level: np.ndarray = None          # per index of net.nodes (UNASSIGNED = none)
    node_ids: np.ndarray = None

    def layer_of(self, node_id: int) -> Optional[int]:
        i = np.searchsorted(self.node_ids, node_id)
        if i >= len(self.node_ids) or self.node_ids[i] != node_id:
            return None
        lv = int(self.level[i])
        return None if lv == _lib.UNASSIGNED else lv

    def assigned_count(self) -> int:
        return sum(len(l) for l in self.layers)


def depth(assignment: LayerAssignment) -> int:
    """segmentation.cpp:103-105."""
    return len(assignment.layers)


def unassigned_outputs(net: Network, assignment: LayerAssignment) -> list:
    """segmentation.cpp:107-112."""
    return [int(o) for o in net.outputs if assignment.layer_of(int(o)) is None]


@dataclass
class LayeredLayout:
    """LayeredLayout (layout.hpp:27-37) in CSR form."""
    total_layers: int
    layer_offsets: np.ndarray
    node_ids: np.ndarray
    row_ptr: np.ndarray
    in_nodes: np.ndarray
    in_weights: np.ndarray
    input_order: np.ndarray
    dropped_connections: int
    id_bound: int
    outputs: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))

    def __post_init__(self):
        self.layer_offsets = _u32(self.layer_offsets)
        self.node_ids = _u32(self.node_ids)
        self.row_ptr = np.ascontiguousarray(np.asarray(self.row_ptr, dtype=np.uint64))
        self.in_nodes = _u32(self.in_nodes)
        self.in_weights = _f32(self.in_weights)
        self.input_order = _u32(self.input_order)
        self.outputs = _u32(self.outputs)

    @property
    def nodes_per_layer(self) -> np.ndarray:
        return np.diff(self.layer_offsets).astype(np.uint32)

    def node_count(self) -> int:
        return len(self.node_ids)

    @property
    def node_layer(self) -> np.ndarray:
        return np.repeat(np.arange(self.total_layers, dtype=np.uint32), self.nodes_per_layer)

    @property
    def is_sensor(self) -> np.ndarray:
        return self.node_layer == 0

    def row(self, k: int):
        b, e = int(self.row_ptr[k]), int(self.row_ptr[k + 1])
        return self.in_nodes[b:e], self.in_weights[b:e]

    def desc(self) -> _lib.LayoutDesc:
        d = _lib.LayoutDesc()
        d.total_layers = self.total_layers
        d.layer_offsets = _lib.ptr(self.layer_offsets, C.c_uint32)
        d.node_count = len(self.node_ids)
        d.node_ids = _lib.ptr(self.node_ids, C.c_uint32)
        d.row_ptr = _lib.ptr(self.row_ptr, C.c_uint64)
        d.in_nodes = _lib.ptr(self.in_nodes, C.c_uint32)
        d.in_weights = _lib.ptr(self.in_weights, C.c_float)
        d.n_inputs = len(self.input_order)
        d.input_order = _lib.ptr(self.input_order, C.c_uint32)
        d.id_bound = self.id_bound
        d.n_outputs = len(self.outputs)
        d.outputs = _lib.ptr(self.outputs, C.c_uint32)
        return d


def layer_slice_bounds(layout: LayeredLayout, layer: int):
    """layout.cpp:85-91."""
    if layer >= layout.total_layers:
        raise LayerOutOfRange(f"layer {layer} out of range, total layers {layout.total_layers}")
    return int(layout.layer_offsets[layer]), int(layout.layer_offsets[layer + 1] -
                                                 layout.layer_offsets[layer])


def max_layer_width(layout: LayeredLayout) -> int:
    """eval.cpp:89-94."""
    return int(layout.nodes_per_layer.max()) if layout.total_layers else 0


@dataclass
class ActivationState:
    """ActivationState (eval.hpp:14-17): id-indexed inputs and op values."""
    inputs: np.ndarray
    outputs: np.ndarray


class Backend(enum.Enum):
    HostParallel = 0
    DeviceCompute = 1


@dataclass
class ParallelConfig:
    """ParallelConfig (eval.hpp:19-27)."""
    workers: int = 0
    backend: Backend = Backend.HostParallel
    node_hook: Optional[Callable[[int], None]] = None
    device: int = 0


# --- device handle ------------------------------------------------------------
class Device:
    """One asnn_dev (CUDA device + stream)."""

    _default: dict = {}
    _lock = threading.Lock()

    def __init__(self, index: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        rc = self.lib.asnn_dev_open(index, C.byref(h))
        if rc:
            raise BackendUnavailable(f"no CUDA device {index} for the device-compute backend")
        self.h = h
        self.index = index
        self.sweep_mode = int(os.environ.get("ASNN_SWEEP_MODE", "0") or 0) % 5

    @classmethod
    def get(cls, index: int = 0) -> "Device":
        with cls._lock:
            if index not in cls._default:
                cls._default[index] = Device(index)
            return cls._default[index]

    def check(self, rc: int):
        if rc:
            _raise(rc, (self.lib.asnn_dev_last_error(self.h) or b"").decode())

    def set_stream(self, stream_ptr: Optional[int]):
        self.check(self.lib.asnn_dev_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def synchronize(self):
        self.check(self.lib.asnn_dev_synchronize(self.h))

    def set_sweep_mode(self, mode: int):
        """0 automatic, 1 one launch per level (heavy rows split across levels
        where eligible), 2 one CTA per (network, slice), 3 one launch per level
        with whole rows only."""
        self.check(self.lib.asnn_dev_set_sweep_mode(self.h, int(mode)))
        self.sweep_mode = int(mode)

    def set_heavy_threshold(self, min_in_degree: Optional[int]):
        """Rows above this in-degree use the streamed heavy kernel (None = off)."""
        v = 0xFFFFFFFF if min_in_degree is None else int(min_in_degree)
        self.check(self.lib.asnn_dev_set_heavy_threshold(self.h, v))

    def timings(self) -> dict:
        t = _lib.Timings()
        self.check(self.lib.asnn_dev_last_timings(self.h, C.byref(t)))
        return {n: getattr(t, n) for n, _ in _lib.Timings._fields_}

    def close(self):
        if self.h:
            self.lib.asnn_dev_close(self.h)
            self.h = None


def device_count() -> int:
    n = C.c_int(0)
    _lib.load().asnn_dev_device_count(C.byref(n))
    return n.value


# --- preprocessing on the device ----------------------------------------------
def compute_required(net: Network, device: int = 0) -> RequiredSet:
    """network.cpp:222-255, as a reverse-frontier BFS on the GPU."""
    dev = Device.get(device)
    mask = np.zeros(len(net.nodes), dtype=np.uint8)
    d = net.desc()
    dev.check(dev.lib.asnn_dev_compute_required(dev.h, C.byref(d), _lib.ptr(mask, C.c_uint8)))
    return RequiredSet(net.nodes[mask.astype(bool)])


def segment(net: Network, required: Optional[RequiredSet] = None, device: int = 0) -> LayerAssignment:
    """segmentation.cpp:20-101, as a Kahn pass on the GPU (levels bit-exact)."""
    dev = Device.get(device)
    level = np.empty(len(net.nodes), dtype=np.uint32)
    n_layers = C.c_uint32(0)
    d = net.desc()
    mask = None
    if required is not None:
        mask = np.isin(net.nodes, required.members).astype(np.uint8)
    dev.check(dev.lib.asnn_dev_segment(dev.h, C.byref(d), _lib.ptr(mask, C.c_uint8),
                                       _lib.ptr(level, C.c_uint32), C.byref(n_layers)))
    return _assignment_from_levels(net, level, n_layers.value)


def _assignment_from_levels(net: Network, level: np.ndarray, n_layers: int) -> LayerAssignment:
    assigned = level != _lib.UNASSIGNED
    order = np.lexsort((net.nodes[assigned], level[assigned]))
    ids = net.nodes[assigned][order]
    lv = level[assigned][order]
    bounds = np.searchsorted(lv, np.arange(n_layers + 1))
    layers = [ids[bounds[l]:bounds[l + 1]] for l in range(n_layers)]
    return LayerAssignment(layers, net.nodes[~assigned], level, net.nodes)


class DeviceLayout:
    """A device-resident level-sorted CSR (asnn_dev_layout): build once,
    activate many batches.  The amortised fast path of the engine."""

    def __init__(self, dev: Device, handle: C.c_void_p):
        self.dev = dev
        self.h = handle
        self._info = None

    # construction -----------------------------------------------------------
    @classmethod
    def from_network(cls, net: Network, device: int = 0) -> "DeviceLayout":
        """compute_required + segment + flatten on the GPU."""
        dev = Device.get(device)
        h = C.c_void_p()
        d = net.desc()
        dev.check(dev.lib.asnn_dev_build_layout(dev.h, C.byref(d), C.byref(h)))
        return cls(dev, h)

    @classmethod
    def from_text(cls, text, device: int = 0) -> "DeviceLayout":
        """load -> levels entirely on the GPU: parse_network + validate +
        compute_required + segment + flatten of an `asnn 1` text."""
        if isinstance(text, str):
            text = text.encode()
        dev = Device.get(device)
        h = C.c_void_p()
        line = C.c_uint32(0)
        rc = dev.lib.asnn_dev_load_layout(dev.h, text, len(text), C.byref(h), C.byref(line))
        if rc == _lib.ASNN_E_PARSE:
            raise ParseError(dev.lib.asnn_dev_last_error(dev.h).decode(), line.value)
        dev.check(rc)
        return cls(dev, h)

    @classmethod
    def from_population(cls, nets: Sequence[Network], device: int = 0) -> "DeviceLayout":
        dev = Device.get(device)
        descs = (_lib.NetworkDesc * len(nets))(*[n.desc() for n in nets])
        h = C.c_void_p()
        dev.check(dev.lib.asnn_dev_build_population(dev.h, len(nets), descs, C.byref(h)))
        return cls(dev, h)

    @classmethod
    def from_layout(cls, layout: LayeredLayout, device: int = 0) -> "DeviceLayout":
        dev = Device.get(device)
        h = C.c_void_p()
        d = layout.desc()
        dev.check(dev.lib.asnn_dev_upload_layout(dev.h, C.byref(d), C.byref(h)))
        return cls(dev, h)

    def free(self):
        if self.h:
            srv = getattr(self, "_server", None)
            if srv is not None and srv.h:
                srv.h = None  # asnn_dev_free_layout stops it
            self.dev.lib.asnn_dev_free_layout(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    # queries ------------------------------------------------------------------
    def info(self, net_index: Optional[int] = None) -> dict:
        i = _lib.LayoutInfo()
        if net_index is None:
            self.dev.check(self.dev.lib.asnn_dev_layout_info(self.h, C.byref(i)))
        else:
            self.dev.check(self.dev.lib.asnn_dev_network_info(self.h, net_index, C.byref(i)))
        return {n: getattr(i, n) for n, _ in _lib.LayoutInfo._fields_}

    def layer_slice(self, layer: int):
        s, c = C.c_uint32(), C.c_uint32()
        self.dev.check(self.dev.lib.asnn_dev_layer_slice(self.h, layer, C.byref(s), C.byref(c)))
        return s.value, c.value

    def download(self, net_index: int = 0) -> LayeredLayout:
        """The flattened layout back in the reference's form (flatten parity)."""
        inf = self.info(net_index)
        L, N, E = inf["total_layers"], inf["node_count"], inf["edge_count"]
        lo = np.zeros(L + 1, np.uint32)
        ids = np.zeros(N, np.uint32)
        rp = np.zeros(N + 1, np.uint64)
        src = np.zeros(E, np.uint32)
        w = np.zeros(E, np.float32)
        io = np.zeros(inf["n_inputs"], np.uint32)
        self.dev.check(self.dev.lib.asnn_dev_layout_download(
            self.h, net_index, _lib.ptr(lo, C.c_uint32), _lib.ptr(ids, C.c_uint32),
            _lib.ptr(rp, C.c_uint64), _lib.ptr(src, C.c_uint32), _lib.ptr(w, C.c_float),
            _lib.ptr(io, C.c_uint32)))
        return LayeredLayout(L, lo, ids, rp, src, w, io, inf["dropped_connections"],
                             inf["id_bound"])

    def plan(self, n_vec: int) -> dict:
        k, b, ce = C.c_uint32(), C.c_uint64(), C.c_uint64()
        self.dev.check(self.dev.lib.asnn_dev_activate_plan(self.h, n_vec, C.byref(k), C.byref(b),
                                                           C.byref(ce)))
        kind = C.c_uint32()
        self.dev.check(self.dev.lib.asnn_dev_sweep_kind(self.h, n_vec, C.byref(kind)))
        return {"kernels": k.value, "alg_bytes": b.value, "conn_evals": ce.value,
                "strategy": ("rows", "segments", "k_cta", "k_chain")[kind.value]}

    def profile(self, x_ptr: int, n_vec: int, out_ptr: int) -> np.ndarray:
        """Per-stage device ms of one sweep (sensors, each level, gather)."""
        k = self.plan(n_vec)["kernels"] + 2 * self.info()["total_layers"] + 2
        ms = np.zeros(k, np.float32)
        n = C.c_uint32()
        self.dev.check(self.dev.lib.asnn_dev_profile_sweep(
            self.h, C.c_void_p(x_ptr), n_vec, C.c_void_p(out_ptr), _lib.ptr(ms, C.c_float),
            C.byref(n)))
        return ms[:n.value]

    # activation ---------------------------------------------------------------
    def activate(self, X: np.ndarray, outputs: bool = True, state: bool = False,
                 n_vec: Optional[int] = None):
        """X: [n_vec][n_inputs] float32 (host) for one network.  For a
        population pass X as [n_networks][n_vec][n_inputs] (or any buffer
        holding each network's [n_vec][n_inputs] block in order) together with
        n_vec.  Returns (out, state): out holds each network's
        [n_vec][n_outputs] block, state each network's [n_vec][id_bound]
        block; for a single network they are shaped [n_vec][...]."""
        X = np.ascontiguousarray(X, dtype=np.float32)
        if n_vec is None:
            if X.ndim == 1:
                X = X[None, :]
            n_vec = X.shape[0]
        inf = self.info() if self._info is None else self._info
        self._info = inf
        out = np.empty((n_vec, inf["n_outputs"]), np.float32) if outputs else None
        st = np.empty((n_vec, inf["id_bound"]), np.float32) if state else None
        self.dev.check(self.dev.lib.asnn_dev_activate(
            self.h, _lib.ptr(X, C.c_float), n_vec, X.size, _lib.ptr(out, C.c_float),
            _lib.ptr(st, C.c_float)))
        return out, st

    def activate_host_ptr(self, x_ptr: int, n_vec: int, n_x: int, out_ptr: int):
        """Host-buffer activation by raw pointers (pinned torch tensors)."""
        rc = self.dev.lib.activate_addr(self.h, x_ptr, n_vec, n_x, out_ptr, None)
        if rc:
            self.dev.check(rc)

    def activate_device(self, x_ptr: int, n_vec: int, out_ptr: int):
        """Device pointers, stream-ordered on the device handle's stream."""
        self.dev.check(self.dev.lib.asnn_dev_activate_device(
            self.h, C.c_void_p(x_ptr), n_vec, C.c_void_p(out_ptr)))

    def serve(self, max_vec: int = 1) -> "Server":
        """Start the resident batch-1 server for this (single-network) layout
        (asnn_dev_server_start, csrc/serve.cuh)."""
        h = C.c_void_p()
        self.dev.check(self.dev.lib.asnn_dev_server_start(self.h, max_vec, C.byref(h)))
        self._server = Server(self, h, max_vec)
        return self._server


class Server:
    """A persistent one-CTA kernel holding one layout in shared memory and
    answering activations through a doorbell in page-locked host memory: no
    launch or stream synchronisation per call.  Use as a context manager or
    call close(); freeing the layout stops it too."""

    def __init__(self, layout: "DeviceLayout", h, max_vec: int):
        self.layout, self.h, self.max_vec = layout, h, max_vec
        inf = layout.info() if layout._info is None else layout._info
        layout._info = inf
        self.n_in, self.n_out = inf["n_inputs"], inf["n_outputs"]

    def activate(self, X: np.ndarray) -> np.ndarray:
        """X: [n_vec][n_inputs] float32 -> outputs [n_vec][n_outputs]."""
        X = np.ascontiguousarray(X, dtype=np.float32)
        if X.ndim == 1:
            X = X[None, :]
        out = np.empty((X.shape[0], self.n_out), np.float32)
        self.layout.dev.check(self.layout.dev.lib.asnn_dev_server_activate(
            self.h, _lib.ptr(X, C.c_float), X.shape[0], X.size, _lib.ptr(out, C.c_float)))
        return out

    def activate_ptr(self, x_ptr: int, n_vec: int, n_x: int, out_ptr: int):
        """Raw host pointers (no per-call ctypes casts)."""
        rc = self.layout.dev.lib.server_activate_addr(self.h, x_ptr, n_vec, n_x, out_ptr)
        if rc:
            self.layout.dev.check(rc)

    def timings(self) -> dict:
        """The last activation: host round trip (us) and device phases (cycles)."""
        ns = C.c_double()
        cyc = (C.c_int64 * 8)()
        self.layout.dev.check(self.layout.dev.lib.asnn_dev_server_timings(self.h, C.byref(ns), cyc))
        return {"round_trip_us": ns.value / 1e3, "sensors_cyc": cyc[0], "layers_cyc": cyc[1],
                "outputs_cyc": cyc[2], "wait_cyc": cyc[3], "dbg": list(cyc[4:8])}

    def close(self):
        if self.h:
            self.layout.dev.lib.asnn_dev_server_stop(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class DeviceGroup:
    """One process driving several GPUs (asnn_group, csrc/group.cu): batch
    sharding over layout replicas, population sharding over network slices,
    the declared outputs all-gathered on the devices (NCCL, or the copy
    engines when a device is listed twice / NCCL is absent)."""

    GATHER = {0: "single device", 1: "nccl", 2: "copy engines"}

    def __init__(self, devices: Sequence[int]):
        self.lib = _lib.load()
        ids = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        rc = self.lib.asnn_group_open(ids, len(devices), C.byref(h))
        if rc:
            _raise(rc, f"cannot open devices {list(devices)}")
        self.h = h
        self.devices = list(devices)

    def check(self, rc: int):
        if rc:
            _raise(rc, (self.lib.asnn_group_last_error(self.h) or b"").decode())

    @property
    def gather(self) -> str:
        n, k = C.c_uint32(), C.c_uint32()
        self.check(self.lib.asnn_group_info(self.h, C.byref(n), C.byref(k)))
        return self.GATHER[k.value]

    @property
    def gather_note(self) -> str:
        return (self.lib.asnn_group_gather_note(self.h) or b"").decode()

    def set_sweep_mode(self, mode: int):
        for i in range(len(self.devices)):
            self.lib.asnn_dev_set_sweep_mode(self.lib.asnn_group_device(self.h, i), int(mode))

    def layout(self, net: Network) -> "GroupLayout":
        h = C.c_void_p()
        d = net.desc()
        self.check(self.lib.asnn_group_build_layout(self.h, C.byref(d), C.byref(h)))
        return GroupLayout(self, h, [net])

    def upload(self, layout: LayeredLayout) -> "GroupLayout":
        h = C.c_void_p()
        d = layout.desc()
        self.check(self.lib.asnn_group_upload_layout(self.h, C.byref(d), C.byref(h)))
        return GroupLayout(self, h, None)

    def population(self, nets: Sequence[Network]) -> "GroupLayout":
        descs = (_lib.NetworkDesc * len(nets))(*[n.desc() for n in nets])
        h = C.c_void_p()
        self.check(self.lib.asnn_group_build_population(self.h, len(nets), descs, C.byref(h)))
        return GroupLayout(self, h, list(nets), population=True)

    def close(self):
        if self.h:
            self.lib.asnn_group_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GroupLayout:
    """A layout sharded over a DeviceGroup (asnn_group_layout)."""

    def __init__(self, grp: DeviceGroup, h, nets, population: bool = False):
        self.grp, self.h, self.nets, self.population = grp, h, nets, population
        self._staged = 0

    def _totals(self):
        m = C.c_void_p()
        n_in = n_out = idb = 0
        for i in range(len(self.grp.devices)):
            self.grp.check(self.grp.lib.asnn_group_layout_member(self.h, i, C.byref(m)))
            if not m.value:
                continue
            inf = _lib.LayoutInfo()
            self.grp.check(self.grp.lib.asnn_dev_layout_info(m, C.byref(inf)))
            if not self.population:
                return inf.n_inputs, inf.n_outputs, inf.id_bound
            n_in, n_out, idb = n_in + inf.n_inputs, n_out + inf.n_outputs, idb + inf.id_bound
        return n_in, n_out, idb

    def shard(self, i: int, n_vec: int) -> dict:
        v = C.c_uint32()
        xo, xc, oo, oc = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.grp.check(self.grp.lib.asnn_group_shard(self.h, i, n_vec, C.byref(v), C.byref(xo),
                                                     C.byref(xc), C.byref(oo), C.byref(oc)))
        return dict(vecs=v.value, x_off=xo.value, x_count=xc.value, out_off=oo.value,
                    out_count=oc.value)

    def activate(self, X: np.ndarray, n_vec: Optional[int] = None, state: bool = False):
        """Like DeviceLayout.activate: (out, state) over the whole batch /
        population, computed across the group's devices."""
        X = np.ascontiguousarray(X, dtype=np.float32)
        if n_vec is None:
            X = X[None, :] if X.ndim == 1 else X
            n_vec = X.shape[0]
        n_in, n_out, idb = self._totals()
        out = np.empty(n_vec * n_out, np.float32)
        st = np.empty(n_vec * idb, np.float32) if state else None
        self.grp.check(self.grp.lib.asnn_group_activate(
            self.h, _lib.ptr(X, C.c_float), n_vec, X.size, _lib.ptr(out, C.c_float),
            _lib.ptr(st, C.c_float)))
        if not self.population:
            out = out.reshape(n_vec, n_out)
            st = st.reshape(n_vec, idb) if st is not None else None
        return out, st

    def stage(self, X: np.ndarray, n_vec: int):
        X = np.ascontiguousarray(X, dtype=np.float32)
        self.grp.check(self.grp.lib.asnn_group_stage_inputs(self.h, _lib.ptr(X, C.c_float), n_vec,
                                                            X.size))
        self._staged = n_vec

    def sweep(self, repeats: int = 1) -> float:
        """Resident sweeps + gathers of the staged batch: device ms per sweep
        (max over the group's devices)."""
        ms = C.c_float()
        self.grp.check(self.grp.lib.asnn_group_sweep(self.h, repeats, C.byref(ms)))
        return ms.value

    def read_outputs(self) -> np.ndarray:
        _, n_out, _ = self._totals()
        out = np.empty(self._staged * n_out, np.float32)
        self.grp.check(self.grp.lib.asnn_group_read_outputs(self.h, _lib.ptr(out, C.c_float)))
        return out

    def free(self):
        if self.h:
            self.grp.lib.asnn_group_free_layout(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def comm_unique_id() -> bytes:
    """128-byte NCCL id for a one-process-per-GPU job (rank 0 makes it, the
    launcher's store distributes it; Device.comm_init joins)."""
    buf = (C.c_uint8 * 128)()
    rc = _lib.load().asnn_comm_unique_id(buf)
    if rc:
        _raise(rc, "NCCL is not available")
    return bytes(buf)


def _device_comm_init(self, uid: bytes, n_ranks: int, rank: int):
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    self.check(self.lib.asnn_dev_comm_init(self.h, buf, n_ranks, rank))


def _device_allgather(self, send_ptr: int, recv_ptr: int, counts: Sequence[int]):
    """Stream-ordered all-gather of float slices (counts per rank, rank order)."""
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    self.check(self.lib.asnn_dev_allgather(self.h, C.c_void_p(send_ptr), C.c_void_p(recv_ptr),
                                           _lib.ptr(c, C.c_uint64)))


Device.comm_init = _device_comm_init
Device.allgather = _device_allgather


def flatten(net: Network, assignment: Optional[LayerAssignment] = None,
            device: int = 0) -> LayeredLayout:
    """layout.cpp:12-83 on the GPU.  The device layout is rebuilt from the
    network; when an assignment is passed its levels must agree (they are
    the device's own segment() result in every caller of this mirror)."""
    if assignment is not None:
        missing = unassigned_outputs(net, assignment)
        if missing:
            raise OutputUnreachable("unassigned output node(s): " + " ".join(map(str, missing)))
    dl = DeviceLayout.from_network(net, device)
    try:
        lay = dl.download(0)
    finally:
        dl.free()
    lay.outputs = _u32(net.outputs)
    return lay


def eval_parallel(layout: LayeredLayout, input_values, cfg: ParallelConfig = ParallelConfig()
                  ) -> ActivationState:
    """eval.cpp:49-80.  Backend.DeviceCompute uploads the layout on every call
    (the reference mutates layouts in place between evaluations,
    asnn_main.cpp:264-278) and returns the id-indexed state."""
    if cfg.backend != Backend.DeviceCompute:
        raise BackendUnavailable("this engine implements Backend::DeviceCompute only; "
                                 "HostParallel is the reference's CPU evaluator")
    if cfg.node_hook is not None:
        raise BackendUnavailable("node_hook cannot run per node on the device backend")
    x = _f32(input_values)
    if len(x) != len(layout.input_order):
        raise InputArityMismatch(f"expected {len(layout.input_order)} input values, got {len(x)}")
    if Device.get(cfg.device).sweep_mode:
        # an explicitly chosen sweep strategy runs on an uploaded layout
        return eval_parallel_batch(layout, x[None, :], cfg)[0]
    inputs = np.zeros(layout.id_bound, np.float32)
    inputs[layout.input_order] = x   # make_state, eval.cpp:32-33 (last duplicate wins)
    return ActivationState(inputs, eval_once(layout, x, cfg.device))


def eval_once(layout: LayeredLayout, x, device: int = 0) -> np.ndarray:
    """One eval_parallel call on a layout that exists for this call only
    (asnn_dev_eval_layout, once.cu): returns state.outputs [id_bound]."""
    dev = Device.get(device)
    x = _f32(x)
    out = np.empty(layout.id_bound, np.float32)
    d = layout.desc()
    dev.check(dev.lib.asnn_dev_eval_layout(dev.h, C.byref(d), _lib.ptr(x, C.c_float), len(x),
                                           _lib.ptr(out, C.c_float)))
    return out


class EvalBuffer:
    """asnn_eval_buf: page-locked staging the caller writes a layout into, then
    one device call (once.cu).  `stage` returns numpy views of the staged arrays;
    they stay valid until the next `stage` (which may reallocate) or `free`.
    One buffer per thread."""

    def __init__(self, device: int = 0):
        self.dev = Device.get(device)
        self.h = C.c_void_p()
        self.dev.check(self.dev.lib.asnn_eval_buf_create(self.dev.h, C.byref(self.h)))

    def stage(self, total_layers: int, node_count: int, sensor_count: int, id_bound: int,
              edge_count: int) -> dict:
        d = _lib.EvalDims(total_layers, node_count, sensor_count, id_bound, edge_count)
        st = _lib.EvalStage()
        self.dev.check(self.dev.lib.asnn_eval_buf_stage(self.h, C.byref(d), C.byref(st)))
        self.id_bound = id_bound

        def view(p, n, t):
            return np.ctypeslib.as_array(p, shape=(max(n, 1),))[:n].view(t) if n else np.zeros(0, t)
        return {"layer_offsets": view(st.layer_offsets, total_layers + 1, np.uint32),
                "node_ids": view(st.node_ids, node_count, np.uint32),
                "row_ptr": view(st.row_ptr, node_count + 1, np.uint32),
                "in_nodes": view(st.in_nodes, edge_count, np.uint32),
                "in_weights": view(st.in_weights, edge_count, np.float32),
                "sensor_inputs": view(st.sensor_inputs, sensor_count, np.float32)}

    def stage_layout(self, layout: LayeredLayout, x) -> None:
        x = _f32(x)
        n = len(layout.node_ids)
        ns = int(layout.layer_offsets[1]) if layout.total_layers else 0
        a = self.stage(layout.total_layers, n, ns, layout.id_bound, int(layout.row_ptr[-1]) if n else 0)
        a["layer_offsets"][:] = layout.layer_offsets
        a["node_ids"][:] = layout.node_ids
        a["row_ptr"][:] = layout.row_ptr
        a["in_nodes"][:] = layout.in_nodes
        a["in_weights"][:] = layout.in_weights
        inputs = np.zeros(layout.id_bound, np.float32)
        inputs[layout.input_order] = x
        a["sensor_inputs"][:] = inputs[layout.node_ids[:ns]]

    def run(self) -> np.ndarray:
        out = np.empty(self.id_bound, np.float32)
        self.dev.check(self.dev.lib.asnn_eval_buf_run(self.h, _lib.ptr(out, C.c_float)))
        return out

    @property
    def mode(self) -> int:
        m = C.c_uint32(0)
        self.dev.check(self.dev.lib.asnn_eval_buf_mode(self.h, C.byref(m)))
        return m.value

    def free(self):
        if self.h:
            self.dev.lib.asnn_eval_buf_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def eval_parallel_batch(layout: LayeredLayout, X, cfg: ParallelConfig = ParallelConfig(
        backend=Backend.DeviceCompute)) -> list:
    """eval_parallel over a batch of input vectors X [n_vec][n_in]."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    if X.ndim != 2 or X.shape[1] != len(layout.input_order):
        raise InputArityMismatch(
            f"expected {len(layout.input_order)} input values per vector, got shape {X.shape}")
    dl = DeviceLayout.from_layout(layout, cfg.device)
    try:
        _, st = dl.activate(X, outputs=False, state=True)
    finally:
        dl.free()
    res = []
    for v in range(X.shape[0]):
        inputs = np.zeros(layout.id_bound, np.float32)
        inputs[layout.input_order] = X[v]   # make_state, eval.cpp:32-33 (last duplicate wins)
        res.append(ActivationState(inputs, st[v]))
    return res


def read_outputs(state: ActivationState, net: Network) -> np.ndarray:
    """eval.cpp:82-87."""
    return state.outputs[net.outputs]


# --- corpora (netgen.cpp:71-157 and the config shapes) ---------------------------
@dataclass
class GenSpec:
    """GenSpec (netgen.hpp:13-22)."""
    input_count: int = 1
    output_count: int = 1
    hidden_count: int = 0
    connection_count: int = 0
    target_depth: int = 2
    weight_min: float = -1.0
    weight_max: float = 1.0
    seed: int = 0


def _corpus_to_network(lib, h) -> Network:
    d = _lib.NetworkDesc()
    lib.asnn_corpus_desc(h, C.byref(d))

    def arr(p, n, dt):
        if n == 0:
            return np.zeros(0, dt)
        return np.ctypeslib.as_array(p, shape=(n,)).copy()
    net = Network(arr(d.nodes, d.n_nodes, np.uint32), arr(d.inputs, d.n_inputs, np.uint32),
                  arr(d.outputs, d.n_outputs, np.uint32), arr(d.source, d.n_connections, np.uint32),
                  arr(d.target, d.n_connections, np.uint32), arr(d.weight, d.n_connections, np.float32))
    lib.asnn_corpus_free(h)
    return net


def generate(spec: GenSpec) -> Network:
    """netgen.cpp:71-157, byte-identical to the reference for the same spec."""
    lib = _lib.load()
    h = C.c_void_p()
    rc = lib.asnn_gen_reference(spec.input_count, spec.output_count, spec.hidden_count,
                                spec.connection_count, spec.target_depth, spec.weight_min,
                                spec.weight_max, spec.seed & 0xFFFFFFFFFFFFFFFF, C.byref(h))
    if rc:
        _raise(rc, "infeasible GenSpec")
    return _corpus_to_network(lib, h)


# --- io.hpp:23-31: loading on the device (csrc/parse.cu) ------------------------
def parse_network(text, device: int = 0) -> Network:
    """parse_network (io.cpp:83-156) + validate (network.cpp:151-216) on the
    device: raises ParseError (with .line) or ValidationError with the
    reference's messages."""
    if isinstance(text, str):
        text = text.encode()
    dev = Device.get(device)
    h = C.c_void_p()
    line = C.c_uint32(0)
    rc = dev.lib.asnn_dev_parse_network(dev.h, text, len(text), C.byref(h), C.byref(line))
    if rc == _lib.ASNN_E_PARSE:
        raise ParseError(dev.lib.asnn_dev_last_error(dev.h).decode(), line.value)
    if rc:
        _raise(rc, dev.lib.asnn_dev_last_error(dev.h).decode())
    return _corpus_to_network(dev.lib, h)


def validate(net: Network, device: int = 0) -> list:
    """validate (network.cpp:151-216) on the device: the ValidationReport's
    messages in the reference's order ([] = valid)."""
    dev = Device.get(device)
    buf = C.create_string_buffer(1 << 20)
    n = C.c_uint32(0)
    d = net.desc()
    dev.check(dev.lib.asnn_dev_validate(dev.h, C.byref(d), buf, len(buf), C.byref(n)))
    return buf.value.decode().split("\n") if n.value else []


def normalize(net: Network, device: int = 0) -> Network:
    """normalize (network.cpp:69-85) on the device: ids -> dense positions."""
    dev = Device.get(device)
    h = C.c_void_p()
    d = net.desc()
    dev.check(dev.lib.asnn_dev_normalize(dev.h, C.byref(d), C.byref(h)))
    return _corpus_to_network(dev.lib, h)


def read_network(path, device: int = 0) -> Network:
    """read_network (io.cpp:167-173): the file's bytes through parse_network."""
    dev = Device.get(device)
    h = C.c_void_p()
    line = C.c_uint32(0)
    rc = dev.lib.asnn_dev_read_network(dev.h, str(path).encode(), C.byref(h), C.byref(line))
    if rc == _lib.ASNN_E_PARSE:
        raise ParseError(dev.lib.asnn_dev_last_error(dev.h).decode(), line.value)
    if rc:
        _raise(rc, dev.lib.asnn_dev_last_error(dev.h).decode())
    return _corpus_to_network(dev.lib, h)


def max_connections(spec: GenSpec) -> int:
    """netgen.cpp:63-69."""
    return int(_lib.load().asnn_gen_max_connections(spec.input_count, spec.output_count,
                                                    spec.hidden_count, spec.target_depth))


def generate_mlp(layers: int, width: int, p: float, seed: int) -> Network:
    lib = _lib.load()
    h = C.c_void_p()
    rc = lib.asnn_gen_mlp(layers, width, p, seed, C.byref(h))
    if rc:
        _raise(rc, "bad mlp spec")
    return _corpus_to_network(lib, h)


def generate_powerlaw(n_nodes: int, bands: int, n_inputs: int, n_outputs: int, target_edges: int,
                      alpha: float, seed: int) -> Network:
    lib = _lib.load()
    h = C.c_void_p()
    rc = lib.asnn_gen_powerlaw(n_nodes, bands, n_inputs, n_outputs, target_edges, alpha, seed,
                               C.byref(h))
    if rc:
        _raise(rc, "bad power-law spec")
    return _corpus_to_network(lib, h)


def device_generate_mlp(layers: int, width: int, p: float, seed: int, device: int = 0) -> Network:
    """generate_mlp on the GPU (csrc/gen.cu), byte-identical to the host one."""
    dev = Device.get(device)
    h = C.c_void_p()
    dev.check(dev.lib.asnn_dev_gen_mlp(dev.h, layers, width, p, seed, C.byref(h)))
    return _corpus_to_network(dev.lib, h)


def device_generate_powerlaw(n_nodes: int, bands: int, n_inputs: int, n_outputs: int, target_edges: int,
                             alpha: float, seed: int, device: int = 0) -> Network:
    """generate_powerlaw on the GPU (csrc/gen.cu), byte-identical to the host one."""
    dev = Device.get(device)
    h = C.c_void_p()
    dev.check(dev.lib.asnn_dev_gen_powerlaw(dev.h, n_nodes, bands, n_inputs, n_outputs, target_edges, alpha,
                                            seed, C.byref(h)))
    return _corpus_to_network(dev.lib, h)


def _gen_layout_mlp(cls, layers: int, width: int, p: float, seed: int, device: int = 0):
    dev = Device.get(device)
    h = C.c_void_p()
    dev.check(dev.lib.asnn_dev_gen_mlp_layout(dev.h, layers, width, p, seed, C.byref(h)))
    return cls(dev, h)


def _gen_layout_powerlaw(cls, n_nodes: int, bands: int, n_inputs: int, n_outputs: int, target_edges: int,
                         alpha: float, seed: int, device: int = 0):
    dev = Device.get(device)
    h = C.c_void_p()
    dev.check(dev.lib.asnn_dev_gen_powerlaw_layout(dev.h, n_nodes, bands, n_inputs, n_outputs, target_edges,
                                                   alpha, seed, C.byref(h)))
    return cls(dev, h)


# DeviceLayout.generated_mlp / generated_powerlaw: generate + levels on the GPU
DeviceLayout.generated_mlp = classmethod(_gen_layout_mlp)
DeviceLayout.generated_powerlaw = classmethod(_gen_layout_powerlaw)


class SplitMix64:
    """rng.hpp:10-38 (for seeding corpora and inputs exactly like the reference)."""
    M = 0xFFFFFFFFFFFFFFFF

    def __init__(self, seed: int):
        self.s = seed & self.M

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & self.M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def bounded(self, n: int) -> int:
        threshold = ((1 << 64) - n) % n
        while True:
            r = self.next()
            if r >= threshold:
                return r % n

    def uniform01(self) -> float:
        return (self.next() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        lo32 = float(np.float32(lo))
        return float(np.float32(lo32 + self.uniform01() * (float(np.float32(hi)) - lo32)))


def random_spec(rng: SplitMix64, min_conn: int, max_conn: int) -> GenSpec:
    """test_helpers.hpp:111-131 (seeded feasible specs for property tests)."""
    spec = GenSpec()
    spec.seed = rng.next()
    spec.connection_count = min_conn + rng.bounded(max_conn - min_conn + 1)
    spec.input_count = 1 + rng.bounded(6)
    spec.output_count = 1 + rng.bounded(4)
    spec.target_depth = 3 + rng.bounded(10)
    ceiling = spec.connection_count - spec.output_count if spec.connection_count > spec.output_count else 0
    hidden = max(spec.target_depth - 2, spec.connection_count // 8)
    hidden = min(hidden, ceiling)
    spec.hidden_count = hidden
    while max_connections(spec) < spec.connection_count and hidden < ceiling:
        hidden = min(hidden * 2 + 1, ceiling)
        spec.hidden_count = hidden
    return spec


def corpus_spec(connections: int, depth: int, inputs: int, outputs: int, seed: int) -> GenSpec:
    """make_corpus_spec (asnn_main.cpp:115-135), shared by verify and bench."""
    spec = GenSpec(input_count=inputs, output_count=outputs, connection_count=connections,
                   target_depth=depth, seed=seed)
    if depth > 2:
        ceiling = connections - outputs if connections > outputs else 0
        hidden = max(depth - 2, connections // 10)
        hidden = min(hidden, ceiling)
        spec.hidden_count = hidden
        while max_connections(spec) < connections and hidden < ceiling:
            hidden = min(hidden * 2 + 1, ceiling)
            spec.hidden_count = hidden
    return spec
