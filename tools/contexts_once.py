"""One launch of every NEXT-4 context kernel on the stem activation (fp32 batch
256, bf16 batch 1024), for an ncu capture (tools/profile_contexts.sh)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2104_14129_b200 as A
dev = "cuda:0"
for dt in (torch.float32, torch.bfloat16):
    N = 256 if dt == torch.float32 else 1024
    x = torch.relu(torch.randn((N, 64, 112, 112), device=dev)).to(dt)
    mask, _ = A.relu_pack(x)
    A.relu_pack(x, True)
    A.relu_backward(mask, x)
    y, idx = A.maxpool2d(x, 3, 2, 1)
    A.maxpool2d_backward(idx, y, 112, 112, 3, 2, 1)
    torch.cuda.synchronize()
    del x, mask, y, idx
    torch.cuda.empty_cache()
