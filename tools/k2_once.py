"""One K2 launch at batch N (argv[1], default 4096) on seeded log-normal S (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_14129_b200 as A  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = torch.Generator(device="cpu").manual_seed(20260)
S = torch.exp(2.0 * torch.randn(N, generator=g, dtype=torch.float64)).cuda()
for _ in range(3):
    A.allocate_bits(S, 2 * N, 802816)
torch.cuda.synchronize()
