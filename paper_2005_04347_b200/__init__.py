"""paper_2005_04347_b200 -- B200-native activation engine for sparse,
arbitrary-structured neural networks (arXiv:2005.04347 hot path).

The compute lives in libasnn_b200.so (sm_100a CUDA behind the C-ABI of
include/asnn_dev.h); this package is the host-side mirror of the reference
API (see api.py) plus ctypes plumbing.
"""
from .api import (  # noqa: F401
    ActivationState, Backend, BackendUnavailable, Device, DeviceError, DeviceGroup, DeviceLayout, Server,
    GenSpec, GroupLayout, comm_unique_id, device_generate_mlp, device_generate_powerlaw,
    InfeasibleSpec, InputArityMismatch, IoError, LayerAssignment, LayeredLayout, LayerOutOfRange,
    Network, OutputUnreachable, ParallelConfig, ParseError, RequiredSet, SplitMix64, UnassignedOutput,
    ValidationError, compute_required, normalize, parse_network, read_network, validate,
    corpus_spec, depth, device_count, eval_once, EvalBuffer, eval_parallel, eval_parallel_batch, flatten, generate,
    generate_mlp, generate_powerlaw, layer_slice_bounds, make_network, max_connections,
    max_layer_width, random_spec, read_outputs, segment, unassigned_outputs,
)

__all__ = [n for n in dir() if not n.startswith("_")]
