"""INT32 accumulator overflow behaviour of the tcgen05 kind::i8 path:
all -128 inputs, n = 131088 -> exact sum 131088 * 16384 = 2,147,745,792 > 2^31 - 1."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402

m, n, p = 256, 131088, 256
A = torch.full((m, n), -128, dtype=torch.int8, device="cuda")
B = torch.full((n, p), -128, dtype=torch.int8, device="cuda")
for cg in ("1", "2"):
    os.environ["MM_FORCE_CG"] = cg
    C = mm.gemm(A, B)
    mm.sync_check()
    v = np.unique(C.cpu().numpy())
    exact = n * 128 * 128
    wrap = exact - 2**32
    print(f"cg={cg}: values {v.tolist()}; exact {exact}, wrap {wrap}, saturate {2**31 - 1}")
