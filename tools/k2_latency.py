"""K2 latency at N = 256 .. 16384 (bench.py run_k2_latency), standalone."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_14129_b200 as A  # noqa: E402

print(json.dumps(bench.run_k2_latency(A, 802816, torch.device("cuda:0"), torch)))
