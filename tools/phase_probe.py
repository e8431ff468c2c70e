import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2005_04347_b200 as A
from oracle.bind import Ref
ref = Ref()
for c, d in [(1000, 10), (100000, 10), (1000, 100)]:
    rn = ref.generate(A.corpus_spec(c, d, 8, 2, 7)); rn.preprocess(); lay = rn.layout()
    llay = A.LayeredLayout(lay["total_layers"], lay["layer_offsets"], lay["node_ids"], lay["row_ptr"], lay["in_nodes"], lay["in_weights"], lay["input_order"], lay["dropped_connections"], lay["id_bound"])
    x = np.full((1, len(lay["input_order"])), 0.5, np.float32)
    for rep in range(3):
        t0 = time.perf_counter(); dl = A.DeviceLayout.from_layout(llay); t1 = time.perf_counter()
        dl.activate(x, outputs=True); t2 = time.perf_counter()
        dl.activate(x, outputs=True); t3 = time.perf_counter()
        dl.activate(x, outputs=False, state=True); t4 = time.perf_counter()
        dl.free(); t5 = time.perf_counter()
        print(f"c{c}_d{d} rep{rep}: upload {1e3*(t1-t0):.2f} ms, act1 {1e3*(t2-t1):.2f}, act2 {1e3*(t3-t2):.3f}, act_state {1e3*(t4-t3):.2f}, free {1e3*(t5-t4):.2f}")
