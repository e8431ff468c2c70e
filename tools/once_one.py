"""One shape of the reference bench corpus through asnn_eval_buf_run `reps`
times (for ncu launch lists of the once.cu kernels).
  python tools/once_one.py <connections> <depth> [reps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_04347_b200 as A  # noqa: E402

c, d = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
net = A.generate(A.corpus_spec(c, d, 8, 2, 12345))
lay = A.flatten(net)  # device compute_required / segment / flatten, downloaded
buf = A.EvalBuffer()
buf.stage_layout(lay, np.full(len(lay.input_order), 0.5, np.float32))
for _ in range(reps):
    buf.run()
print("mode", buf.mode, "layers", lay.total_layers, "nodes", len(lay.node_ids), "edges", int(lay.row_ptr[-1]))
