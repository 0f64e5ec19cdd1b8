"""Diagnostics: phase clocks of an instrumented K2 build (off[] holds them)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_14129_b200 as A  # noqa: E402

for N in (256, 4096, 16384):
    g = torch.Generator(device="cpu").manual_seed(20260)
    S = torch.exp(2.0 * torch.randn(N, generator=g, dtype=torch.float64)).cuda()
    for _ in range(3):
        bits, off = A.allocate_bits(S, 2 * N, 802816)
    torch.cuda.synchronize()
    o = off.cpu().tolist()
    nt = -o[0]
    print(N, [o[i] for i in range(1, nt)])
