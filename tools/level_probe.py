"""Per-stage device times of one sweep (asnn_dev_profile_sweep) for a corpus
network of the reference's bench recipe at batch B.
Usage: python tools/level_probe.py <connections> <depth> [B]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2005_04347_b200 as A  # noqa: E402

c, d = int(sys.argv[1]), int(sys.argv[2])
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
net = A.generate(A.corpus_spec(c, d, 8, 2, 7))
dl = A.DeviceLayout.from_network(net)
x = torch.rand(B * len(net.inputs), device="cuda")
out = torch.empty(B * len(net.outputs), device="cuda")
for _ in range(3):
    ms = dl.profile(x.data_ptr(), B, out.data_ptr())
inf = dl.info()
print(f"c{c}_d{d} B={B} strategy={dl.plan(B)['strategy']} nodes={inf['node_count']} edges={inf['edge_count']} levels={inf['total_layers']} stages={len(ms)} total_ms={ms.sum():.4f}")
print(" ".join(f"{v * 1e3:.1f}" for v in ms[:40]), "(us)", flush=True)
