"""Extent of the count-pass row lists at config 5 (rows before the first /
after the last list-A row: their CSR offsets are final after pass 1)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2101_08053_b200 import cases as C
from paper_2101_08053_b200.assembly import form

c5 = C.baseline_config(5, nel=2048)
b2d, cfg = C.build_space(None, 2048, 4, curves=c5["curves"])
f, csr = form(b2d, cfg, None, "dwq")
torch.cuda.synchronize()
w = f.work.cpu().numpy()
K = f.K
na, nb = int(w[0]), int(w[1])
A = np.sort(w[2:2 + na]); B = np.sort(w[2 + K: 2 + K + nb])
print("K", K, "nA", na, "nB", nb)
print("A first/last", A[0], A[-1], "fraction before", A[0] / K, "after", (K - 1 - A[-1]) / K)
print("B first/last", B[0], B[-1])
rf = f.rowfast.cpu().numpy()
print("fast rows", int(rf.sum()), "of", K)
indptr = csr.indptr.cpu().numpy()
print("nnz", int(indptr[-1]), "nnz before A0", int(indptr[A[0]]), "after A_last", int(indptr[-1] - indptr[A[-1] + 1]))
