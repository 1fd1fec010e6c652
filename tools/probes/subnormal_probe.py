"""Subnormal handling of the tcgen05 kind::f16 (BF16 -> FP32) path:
(1) subnormal bf16 inputs times 1.0; (2) normal inputs whose products / sums are FP32 subnormals."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_15384_b200 as mm  # noqa: E402


def bf16(bits):
    return torch.from_numpy(np.asarray(bits, np.uint16).view(np.int16)).view(torch.bfloat16).cuda()


n = 128
# (1) A row 0 = subnormal bf16 values (exponent 0), B = identity
sub = np.arange(1, n + 1, dtype=np.uint16) & 0x7F
sub[sub == 0] = 1
A = np.zeros((256, n), np.uint16)
A[0] = sub
I = np.zeros((n, n), np.uint16)
np.fill_diagonal(I, 0x3F80)  # 1.0
C = mm.gemm(bf16(A), bf16(I)).cpu().numpy()
expect = (sub.astype(np.uint32) << 16).view(np.float32)
print("(1) subnormal inputs x 1.0: kept exactly" if np.array_equal(C[0], expect) else
      f"(1) subnormal inputs x 1.0: flushed/changed: {C[0][:8]} vs {expect[:8]}")
# (2) products that are FP32 subnormals: 2^-70 * 2^-70 = 2^-140
A = np.zeros((256, n), np.uint16)
A[0, 0] = 0x1C80  # 2^-70
B = np.zeros((n, 256), np.uint16)
B[0, 0] = 0x1C80
C = mm.gemm(bf16(A), bf16(B)).cpu().numpy()
print(f"(2) 2^-70 * 2^-70: got {C[0,0]!r} (exact 2^-140 = {np.float32(2.0**-140)!r})")
mm.sync_check()
