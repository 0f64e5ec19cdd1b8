"""ReLU context kernels on the stem activation (fp32 batch 256, bf16 batch 1024):
time per call and fraction of the copy bandwidth (read x, write mask [+ y])."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2104_14129_b200 as A
dev = "cuda:0"
for dt in (torch.float32, torch.bfloat16):
    N = 256 if dt == torch.float32 else 1024
    x = torch.randn((N, 64, 112, 112), device=dev).to(dt)
    mask, _ = A.relu_pack(x)
    gy = torch.randn(x.shape, device=dev).to(dt)
    s, E = x.element_size(), x.numel()
    for name, fn, by in (("pack", lambda: A.relu_pack(x), E * s + E / 8),
                         ("pack+y", lambda: A.relu_pack(x, True), 2 * E * s + E / 8),
                         ("bwd", lambda: A.relu_backward(mask, gy), 2 * E * s + E / 8)):
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000); a.record()
        for _ in range(5): fn()
        b.record(); b.synchronize()
        ms = a.elapsed_time(b) / 5
        print(dt, name, round(ms, 3), "ms", round(by / ms / 1e9 / 6.5447, 3))
