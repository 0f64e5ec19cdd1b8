import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2104_14129_b200 as A
dev = "cuda:0"
for dt in (torch.float32, torch.bfloat16):
    N = 256 if dt == torch.float32 else 1024
    x = torch.relu(torch.randn((N, 64, 112, 112), device=dev)).to(dt)
    y, idx = A.maxpool2d(x, 3, 2, 1)
    gy = torch.randn(y.shape, device=dev).to(dt)
    for name, fn in (("fwd", lambda: A.maxpool2d(x, 3, 2, 1)), ("bwd", lambda: A.maxpool2d_backward(idx, gy, 112, 112, 3, 2, 1))):
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000); a.record()
        for _ in range(5): fn()
        b.record(); b.synchronize()
        ms = a.elapsed_time(b) / 5
        s = x.element_size(); E = x.numel(); EO = y.numel()
        by = E * s + EO * (s + 1)
        print(dt, name, round(ms, 3), "ms", round(by / ms / 1e9 / 6.5447, 3))
