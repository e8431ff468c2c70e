"""Per-call host overhead of the activation entry points on config 1 (one
small network, one vector): device-resident call + sync, host-pointer call
(zero-copy, pinned), and the pieces (ctypes, sync) timed separately."""
import ctypes as C
import time

import numpy as np
import torch

import sys
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2005_04347_b200 as A  # noqa: E402


def per_call(fn, n=2000):
    for _ in range(200):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    net = bench.make_network("c1", 1.0)[0]
    dl = A.DeviceLayout.from_network(net)
    info = dl.info()
    x = np.random.default_rng(0).uniform(-2, 2, (1, len(net.inputs))).astype(np.float32)
    x_dev = torch.from_numpy(x.reshape(-1)).cuda()
    out_dev = torch.empty(info["n_outputs"], dtype=torch.float32, device="cuda")
    x_pin = torch.from_numpy(x.reshape(-1)).pin_memory()
    out_pin = torch.empty(info["n_outputs"], dtype=torch.float32).pin_memory()
    lib, h = dl.dev.lib, dl.h
    xp, op = x_pin.data_ptr(), out_pin.data_ptr()
    f32p = C.POINTER(C.c_float)
    xpc, opc = C.cast(C.c_void_p(xp), f32p), C.cast(C.c_void_p(op), f32p)
    r = {}
    r["device call + torch sync"] = per_call(lambda: (dl.activate_device(x_dev.data_ptr(), 1, out_dev.data_ptr()),
                                                      torch.cuda.synchronize()))
    r["host-ptr call (bench e2e)"] = per_call(lambda: dl.activate_host_ptr(xp, 1, x_pin.numel(), op))
    r["host-ptr call, pre-cast ptrs"] = per_call(lambda: lib.asnn_dev_activate(h, xpc, 1, x_pin.numel(), opc, None))
    r["torch.cuda.synchronize alone"] = per_call(torch.cuda.synchronize)
    r["ctypes no-op (asnn_dev_last_error)"] = per_call(lambda: lib.asnn_dev_last_error(dl.dev.h))
    print({k: round(v, 2) for k, v in r.items()})


if __name__ == "__main__":
    main()
