"""Device CRS build (lmpk_csr_from_triplets) vs the reference's host numpy
build on the cfg2 triplets (gen_stencil_3d(200,2), shuffled)."""
import json, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K

a = lm.gen_stencil_3d(200, 2)
r, c, v = a.to_triplets()
p = np.random.default_rng(0).permutation(r.size)
r, c, v = r[p].astype(np.int64), c[p].astype(np.int64), v[p]
t0 = time.perf_counter()
host = lm.CsrMatrix.from_triplets(a.n_rows, r, c, v)
t_host = time.perf_counter() - t0
rd, cd, vd = (torch.from_numpy(x).cuda() for x in (r, c, v))
K.csr_from_triplets(a.n_rows, rd, cd, vd)  # warm (scratch allocation)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    d = K.csr_from_triplets(a.n_rows, rd, cd, vd)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
rp, col, val = d.to_host()
ok = np.array_equal(rp, host.row_ptr) and np.array_equal(col, host.col) and val.tobytes() == host.val.tobytes()
print(json.dumps({"nnz": int(r.size), "host_numpy_s": t_host, "device_s_min": min(ts), "bitwise": bool(ok),
                  "speedup": t_host / min(ts)}))
