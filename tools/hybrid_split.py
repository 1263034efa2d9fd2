import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2510_08230_b200 import gen
from paper_2510_08230_b200 import sparseops as sp
from tools.sweep_configs import timed_spmv
dev = sp.create_device("cuda", 0)
a = gen.powerlaw_csr(dev)
h = sp.hybrid_from_csr(a)
b = sp.dense_from_array(dev, torch.tensor(np.random.default_rng(0).random(a.rows)))
x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
print("hybrid", timed_spmv(h, b, x), "ell part", timed_spmv(h.ell, b, x), "tail nnz", h.coo.nnz, "ell stored", h.ell.stored, "nnz", a.nnz)
t = sp.CooMatrix(dev, h.coo.rows, h.coo.cols, h.coo.row_idxs, h.coo.col_idxs, h.coo.values)
print("tail via csr index", t.kernel, timed_spmv(t, b, x), "segmented", timed_spmv(h.coo, b, x))
