"""GPU vs oracle parity of the NEXT-4 lossless contexts (ReLU 1-bit mask,
P:1388-1395; max-pool 8-bit argmax) through the C ABI.  Integer
and byte outputs (mask, idx) bit-exact; values bit-exact (they are copies,
zeros, or fp32 sums in the oracle's fixed order)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def A():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2104_14129_b200 as A
    return A


def host_bits(t):
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy().view(np.uint32)


def to_oracle(t):
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def _rand(shape, dtype, seed):
    g = torch.Generator(device=DEV).manual_seed(seed)
    x = torch.randn(shape, generator=g, device=DEV)
    x[..., ::7] = 0.0
    return x.to(dtype)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("E", [1, 9, 1023, 1024, 2048 + 5, 4096 * 3, 1 << 20, 3 * (1 << 20) + 77])
def test_relu_pack_and_backward(A, dtype, E):
    x = _rand((E,), dtype, E)
    g = _rand((E,), dtype, E + 1)
    mask, y = A.relu_pack(x, want_y=True)
    mask2, none = A.relu_pack(x)
    gx = A.relu_backward(mask, g)
    torch.cuda.synchronize()
    m_ref, y_ref = O.relu_pack(to_oracle(x), want_y=True)
    assert none is None
    assert np.array_equal(mask.cpu().numpy(), m_ref)
    assert np.array_equal(mask2.cpu().numpy(), m_ref)
    assert np.array_equal(host_bits(y), y_ref.view(host_bits(y).dtype))
    gx_ref = O.relu_backward(m_ref, to_oracle(g))
    assert np.array_equal(host_bits(gx), gx_ref.view(host_bits(gx).dtype))


def test_relu_unaligned_views(A):
    """Views that start off the 32-byte boundary take the scalar path."""
    base = _rand((70001,), torch.float32, 5)
    x = base[3:]
    mask, y = A.relu_pack(x, want_y=True)
    gx = A.relu_backward(mask, base[1:-2])
    torch.cuda.synchronize()
    m_ref, y_ref = O.relu_pack(to_oracle(x), want_y=True)
    assert np.array_equal(mask.cpu().numpy(), m_ref)
    assert np.array_equal(host_bits(y), y_ref.view(np.uint32))
    assert np.array_equal(host_bits(gx), O.relu_backward(m_ref, to_oracle(base[1:-2])).view(np.uint32))


GEOMS = [  # (N, C, H, W, kernel, stride, padding, dilation)
    (2, 3, 112, 112, (3, 3), (2, 2), (1, 1), (1, 1)),
    (2, 3, 13, 15, (3, 3), (2, 2), (1, 1), (1, 1)),   # odd sizes: the 2x2-block edges
    (1, 2, 8, 7, (3, 3), (2, 2), (1, 1), (1, 1)),
    (1, 2, 13, 16, (3, 3), (2, 2), (1, 1), (1, 1)),   # W % 8 == 0: the vector forward
    (2, 3, 1, 8, (3, 3), (2, 2), (1, 1), (1, 1)),
    (1, 2, 6, 24, (3, 3), (2, 2), (1, 1), (1, 1)),
    (1, 3, 7, 32, (3, 3), (2, 2), (1, 1), (1, 1)),
    (1, 1, 2, 3, (3, 3), (2, 2), (1, 1), (1, 1)),
    (2, 5, 13, 17, (2, 2), (2, 2), (0, 0), (1, 1)),
    (1, 4, 15, 15, (3, 3), (1, 1), (1, 1), (2, 2)),
    (3, 2, 9, 11, (2, 3), (1, 2), (1, 1), (1, 1)),
    (1, 2, 32, 32, (16, 16), (16, 16), (0, 0), (1, 1)),
]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("geom", GEOMS)
def test_maxpool_forward_backward(A, dtype, geom):
    """Integer-valued inputs make ties common (first-argmax rule)."""
    N, C, H, W, k, s, p, d = geom
    g = torch.Generator(device=DEV).manual_seed(H * W)
    x = torch.randint(-4, 5, (N, C, H, W), generator=g, device=DEV).to(dtype)
    y, idx = A.maxpool2d(x, k, s, p, d)
    gy = torch.randn(y.shape, generator=g, device=DEV).to(dtype)
    gx = A.maxpool2d_backward(idx, gy, H, W, k, s, p, d)
    torch.cuda.synchronize()
    y_ref, idx_ref = O.maxpool2d_forward(to_oracle(x), k, s, p, d)
    assert np.array_equal(idx.cpu().numpy(), idx_ref)
    assert np.array_equal(host_bits(y), y_ref.view(host_bits(y).dtype))
    gx_ref = O.maxpool2d_backward(idx_ref, to_oracle(gy), H, W, k, s, p, d)
    assert np.array_equal(host_bits(gx), gx_ref.view(host_bits(gx).dtype))
    # forward values also equal PyTorch's max_pool2d (a library routine)
    yt = torch.nn.functional.max_pool2d(x.float(), k, s, p, d)
    assert torch.equal(y.float(), yt)


def test_maxpool_resnet_stem_full_size_exhaustive(A):
    """The ResNet-50 stem max pool at batch 256 (x = bn1/relu output,
    256 x 64 x 112 x 112 fp32) exhaustively: every output, argmax byte and
    input gradient against the oracle (P:574-592 context of the pooling layer);
    the forward also against torch, gradient mass conserved."""
    N, C, H, W = 256, 64, 112, 112
    g = torch.Generator(device=DEV).manual_seed(50)
    x = torch.relu(torch.randn((N, C, H, W), generator=g, device=DEV))
    y, idx = A.maxpool2d(x, 3, 2, 1)
    gy = torch.randn(y.shape, generator=g, device=DEV)
    gx = A.maxpool2d_backward(idx, gy, H, W, 3, 2, 1)
    torch.cuda.synchronize()
    assert torch.equal(y, torch.nn.functional.max_pool2d(x, 3, 2, 1))
    y_ref, idx_ref = O.maxpool2d_forward(to_oracle(x), (3, 3), (2, 2), (1, 1))
    assert np.array_equal(host_bits(y), y_ref.view(np.uint32))
    assert np.array_equal(idx.cpu().numpy(), idx_ref)
    gx_ref = O.maxpool2d_backward(idx_ref, to_oracle(gy), H, W, (3, 3), (2, 2), (1, 1))
    assert np.array_equal(host_bits(gx), gx_ref.view(np.uint32))
    assert torch.allclose(gx.double().sum(), gy.double().sum(), rtol=1e-9, atol=1e-3)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_maxpool_unaligned_views(A, dtype):
    """Inputs one element off the vector alignment take the scalar k3s2 kernels;
    their outputs equal the vector kernels' (aligned inputs) and the oracle's."""
    N, C, H, W = 2, 3, 14, 32
    g = torch.Generator(device=DEV).manual_seed(7)
    buf = torch.randint(-4, 5, (N * C * H * W + 1,), generator=g, device=DEV).to(dtype)
    x_al = buf[:-1].view(N, C, H, W).clone()
    x_un = buf[1:].view(N, C, H, W)
    x_un.copy_(x_al)
    y_a, i_a = A.maxpool2d(x_al, 3, 2, 1)
    y_u, i_u = A.maxpool2d(x_un, 3, 2, 1)
    gbuf = torch.randn(y_a.numel() + 1, generator=g, device=DEV).to(dtype)
    gy_al = gbuf[:-1].view(y_a.shape).clone()
    gy_un = gbuf[1:].view(y_a.shape)
    gy_un.copy_(gy_al)
    gx_a = A.maxpool2d_backward(i_a, gy_al, H, W, 3, 2, 1)
    gx_u = A.maxpool2d_backward(i_a, gy_un, H, W, 3, 2, 1)
    torch.cuda.synchronize()
    assert torch.equal(i_a, i_u) and np.array_equal(host_bits(y_a), host_bits(y_u))
    assert np.array_equal(host_bits(gx_a), host_bits(gx_u))
    y_ref, idx_ref = O.maxpool2d_forward(to_oracle(x_al), (3, 3), (2, 2), (1, 1))
    assert np.array_equal(i_a.cpu().numpy(), idx_ref)
    gx_ref = O.maxpool2d_backward(idx_ref, to_oracle(gy_al), H, W, (3, 3), (2, 2), (1, 1))
    assert np.array_equal(host_bits(gx_a), gx_ref.view(host_bits(gx_a).dtype))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_maxpool_signed_zero_ties(A, dtype):
    """Windows whose maximum is a zero of either sign: the stored value is the
    first zero tap's, bit for bit (the packed bf16 forward's special case)."""
    N, C, H, W = 2, 2, 16, 32
    g = torch.Generator(device=DEV).manual_seed(11)
    choice = torch.randint(0, 3, (N, C, H, W), generator=g, device=DEV)
    x = torch.where(choice == 0, torch.tensor(-0.0, device=DEV),
                    torch.where(choice == 1, torch.tensor(0.0, device=DEV),
                                torch.tensor(-1.0, device=DEV))).to(dtype)
    y, idx = A.maxpool2d(x, 3, 2, 1)
    torch.cuda.synchronize()
    y_ref, idx_ref = O.maxpool2d_forward(to_oracle(x), (3, 3), (2, 2), (1, 1))
    assert np.array_equal(idx.cpu().numpy(), idx_ref)
    assert np.array_equal(host_bits(y), y_ref.view(host_bits(y).dtype))
    neg0 = 0x8000 if dtype == torch.bfloat16 else 0x80000000
    assert (host_bits(y) == neg0).any() and (host_bits(y) == 0).any()  # both signs of zero win
