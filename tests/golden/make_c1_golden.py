"""Writes tests/golden/c1.json from the ORACLE ONLY (never from the CUDA path).

C1 (BASELINE.json configs[0]): one fp32 tensor N=4 x D=1024,
G=256, uniform 2-bit, seed 42, sample_base 0, x from workloads.c1_tensor().
Run: python tests/golden/make_c1_golden.py   (committed output: c1.json)
"""
import hashlib
import importlib.util
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

spec = importlib.util.spec_from_file_location(
    "workloads", os.path.join(ROOT, "paper_2104_14129_b200", "workloads.py"))
W = importlib.util.module_from_spec(spec)
sys.modules["workloads"] = W
spec.loader.exec_module(W)


def main():
    x = W.c1_tensor()
    packed, zmin, scale, off = O.quantize(x, 2, 42, 0)
    out = O.dequantize(packed, zmin, scale, 2, 4, 1024)
    doc = {
        "_source": "oracle/ (ACTNN-Q v1) via tests/golden/make_c1_golden.py; input "
                   "workloads.c1_tensor(); N=4, D=1024, G=256, bits=2, seed=42, sample_base=0",
        "x_sha256": hashlib.sha256(x.tobytes()).hexdigest(),
        "packed_hex": packed.tobytes().hex(),
        "zmin_bits": [int(v) for v in zmin.view(np.uint32).ravel()],
        "scale_bits": [int(v) for v in scale.view(np.uint32).ravel()],
        "dequant_sha256": hashlib.sha256(out.tobytes()).hexdigest(),
    }
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c1.json"), "w") as f:
        json.dump(doc, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
