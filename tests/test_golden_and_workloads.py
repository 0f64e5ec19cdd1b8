"""Regression pins for the committed golden files and the input recipe."""
import hashlib
import importlib.util
import json
import os

import numpy as np

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_spec = importlib.util.spec_from_file_location(
    "actnn_workloads", os.path.join(ROOT, "paper_2104_14129_b200", "workloads.py"))
W = importlib.util.module_from_spec(_spec)
import sys  # noqa: E402
sys.modules["actnn_workloads"] = W
_spec.loader.exec_module(W)


def test_c1_golden_reproduced_by_oracle():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "c1.json")))
    x = W.c1_tensor()
    assert hashlib.sha256(x.tobytes()).hexdigest() == g["x_sha256"]
    packed, zmin, scale, _ = O.quantize(x, 2, 42, 0)
    assert packed.tobytes().hex() == g["packed_hex"]
    assert zmin.view(np.uint32).ravel().tolist() == g["zmin_bits"]
    assert scale.view(np.uint32).ravel().tolist() == g["scale_bits"]
    out = O.dequantize(packed, zmin, scale, 2, 4, 1024)
    assert hashlib.sha256(out.tobytes()).hexdigest() == g["dequant_sha256"]


def test_activation_set_counts():
    """ResNet-50 107 tensors / 21,778,432 elements per sample;
    ResNet-152 311 / 44,658,688; every D is a multiple of G = 256."""
    for depth, (count, elems) in W.expected_counts().items():
        acts = W.resnet_activation_set(depth)
        assert len(acts) == count
        assert sum(a.D for a in acts) == elems
        assert all(a.D % 256 == 0 for a in acts)


def test_synthetic_draw_is_seeded():
    import torch
    a = W.resnet_activation_set(50)[5]
    x1 = W.synth_activation(a, 3, 5)
    x2 = W.synth_activation(a, 3, 5)
    assert torch.equal(x1, x2) and x1.shape == (3, a.D)
    assert (x1 >= 0).all() == a.relu or not a.relu
