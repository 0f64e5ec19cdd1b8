import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2104_14129_b200 as A
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((1, 1024)).astype(np.float32)).cuda()
for b in (4, 8, 3):
    bits, off = A.uniform_bits(1, 1024, b, "cuda")
    p = A.quantize(x, bits, off, 5, 0)
    torch.cuda.synchronize()
    ref = O.quantize(x.cpu().numpy(), b, 5, 0)
    g = p.packed[:32 * b].cpu().numpy()
    cg, _ = O.dequantize_group(g, 256, b, 0, 1)
    cr, _ = O.dequantize_group(ref[0][:32 * b], 256, b, 0, 1)
    print("b", b, "match", np.array_equal(cg, cr))
    print(" gpu", cg[:16]); print(" ref", cr[:16])
