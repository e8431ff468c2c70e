import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2005_04347_b200 as A
net = A.generate(A.GenSpec(16, 4, 980, 10000, 10, -1.0, 1.0, 1))
dl = A.DeviceLayout.from_network(net, device=0)
X = np.random.default_rng(3).uniform(-2, 2, (4, 16)).astype(np.float32)
ref, _ = dl.activate(X)
print("activate ok", flush=True)
srv = dl.serve(max_vec=1)
print("server started", flush=True)
for i in range(4):
    got = srv.activate(X[i:i+1])
    print(i, np.array_equal(got.view(np.uint32), ref[i:i+1].view(np.uint32)), srv.timings(), flush=True)
srv.close()
