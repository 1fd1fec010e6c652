"""The GPU generator (synthgen/synthgen_cuda.cu) must reproduce the host generator bit for
bit: full-matrix checksums of the BASELINE.json config inputs (SURVEY.md §8 c6 values
for the host side are pinned in test_synthgen.py)."""
import json
import os

import numpy as np
import pytest
import torch

import synthgen as sg

pytestmark = pytest.mark.gpu

with open(os.path.join(os.path.dirname(__file__), "golden", "survey_c6.json")) as f:
    C6 = json.load(f)


@pytest.fixture(scope="module")
def sgg(cuda_device):
    from synthgen import gpu
    return gpu


def _np(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def test_f64_configs(sgg):
    for cfg in ("C1", "C2"):
        g = C6[cfg]
        A = sgg.uniform_f64(g["seed"], 1, g["m"], g["n"])
        B = sgg.uniform_f64(g["seed"], 2, g["n"], g["p"])
        assert sg.checksum(_np(A)) == int(g["csA"], 16)
        assert sg.checksum(_np(B)) == int(g["csB"], 16)


def test_i8_config(sgg):
    g = C6["C3"]
    A = sgg.uniform_i8(g["seed"], 1, 4096, 4096)
    assert sg.checksum(_np(A)) == int(g["csA"], 16)


def test_bf16_box_muller_config(sgg):
    """GPU libm log/sin/cos vs glibc: the bf16-rounded values must still agree everywhere."""
    g = C6["C4"]
    A = sgg.normal_bf16(g["seed"], 1, 16384, 16384)
    assert sg.checksum(_np(A), "bf16") == int(g["csA"], 16)
    B = sgg.normal_bf16(g["seed"], 2, 16384, 16384)
    assert sg.checksum(_np(B), "bf16") == int(g["csB"], 16)


def test_exact_int_variants(sgg):
    for K in (3, 9):
        a = _np(sgg.exact_bf16(3, 1, K, 300, 257))
        assert np.array_equal(a, sg.exact_bf16(3, 1, K, 300, 257))
    a = _np(sgg.exact_f64(4, 2, 2049, 123, 77))
    assert np.array_equal(a, sg.exact_f64(4, 2, 2049, 123, 77))
    a = _np(sgg.uniform_f64(9, 1, 1, 1))
    assert a[0, 0] == sg.uniform_f64(9, 1, 1, 1)[0, 0]
