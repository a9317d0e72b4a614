import os, sys, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K
from oracle import levelmpk_oracle as O
N = int(sys.argv[1])
rp, c, v = O.gen_stencil_3d(N); n = rp.shape[0]-1
a = K.DeviceCsr.from_host(rp, c, v)
perm, inv, lp = K.bfs_levels(a, 0); torch.cuda.synchronize()
p = perm.cpu().numpy(); iv = inv.cpu().numpy()
print("perm is permutation:", np.array_equal(np.sort(p), np.arange(n)), "inv ok:", np.array_equal(iv[p], np.arange(n)), flush=True)
t0 = time.time(); op, olp = O.bfs_levels(rp, c, 0, method="keysort"); print("oracle %.1fs" % (time.time()-t0))
print("levels equal:", np.array_equal(lp, olp), "perm equal:", np.array_equal(p, op))
bad = np.flatnonzero(p != op)
print("n bad", bad.size, bad[:10], p[bad[:10]], op[bad[:10]])
b = K.permute_symmetric(a, perm, inv); torch.cuda.synchronize()
hb = b.to_host(); print("col range", hb[1].min(), hb[1].max(), "n", n)
orp, oc, ov = O.permute_symmetric(rp, c, v, op)
print("permute equal:", np.array_equal(hb[0], orp), np.array_equal(hb[1], oc), np.array_equal(hb[2], ov))
