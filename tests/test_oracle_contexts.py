"""Pins of the oracle's NEXT-4 lossless contexts: the ReLU 1-bit mask
(App. B.3: "ReLU layers only take a single bit per dimension to
store, without any approximation") and the max-pool 8-bit argmax (P:1406-1419,
App. B.4: "We use 8 bits per output location").  Pinned by SPEC's worked
examples and by PyTorch's own CPU relu / max_pool2d
forward and autograd backward (library routines), which the compressed
contexts must reproduce bit for bit (they are lossless)."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
F = torch.nn.functional


def bf16_bits(t):
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


# ----------------------------------------------------------------------------- ReLU
def test_relu_spec_examples():
    """input [-1, 2], grad_y [5, 7] -> mask [0, 1], grad_x [0, 7];
    all-negative input -> zero gradient."""
    mask, y = O.relu_pack(np.array([-1, 2], np.float32), want_y=True)
    assert mask.tolist() == [0b10]
    assert y.tolist() == [0.0, 2.0]
    assert O.relu_backward(mask, np.array([5, 7], np.float32)).tolist() == [0.0, 7.0]
    m2, _ = O.relu_pack(-np.arange(1, 20, dtype=np.float32))
    assert not m2.any()
    assert not O.relu_backward(m2, np.ones(19, np.float32)).any()


@pytest.mark.parametrize("E", [1, 7, 8, 9, 1000, 4099])
def test_relu_matches_torch_autograd(E):
    """Lossless: the 1-bit context reproduces torch's relu forward and its
    autograd backward exactly (fp32); 1 bit per element (ceil(E/8) bytes)."""
    rng = np.random.default_rng(E)
    xa = rng.standard_normal(E).astype(np.float32)
    xa[::5] = 0.0
    xa[1::7] = -0.0
    ga = rng.standard_normal(E).astype(np.float32)
    mask, y = O.relu_pack(xa, want_y=True)
    assert mask.nbytes == (E + 7) // 8
    x = torch.from_numpy(xa).requires_grad_(True)
    out = torch.relu(x)
    out.backward(torch.from_numpy(ga))
    assert np.array_equal(y, out.detach().numpy())  # values (+0 == -0)
    gx = O.relu_backward(mask, ga)
    assert np.array_equal(gx.view(np.uint32), x.grad.numpy().view(np.uint32))
    # bit k of the LSB-first stream is x_k > 0
    assert np.array_equal(np.unpackbits(mask, bitorder="little")[:E], (xa > 0).astype(np.uint8))


def test_relu_bf16():
    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.standard_normal(777).astype(np.float32)).to(torch.bfloat16)
    g = torch.from_numpy(rng.standard_normal(777).astype(np.float32)).to(torch.bfloat16)
    mask, y = O.relu_pack(bf16_bits(x), want_y=True)
    assert np.array_equal(y, bf16_bits(torch.where(x > 0, x, torch.zeros_like(x))))
    gx = O.relu_backward(mask, bf16_bits(g))
    assert np.array_equal(gx, bf16_bits(torch.where(x > 0, g, torch.zeros_like(g))))


# ----------------------------------------------------------------------------- max pool
def test_maxpool_spec_example():
    """input [1,3,2,0], kernel 2, stride 2 -> output [3,2], indices
    [1,0]; grad_y [10,20] -> grad_x [0,10,20,0]."""
    x = np.array([1, 3, 2, 0], np.float32).reshape(1, 1, 1, 4)
    y, idx = O.maxpool2d_forward(x, (1, 2), (1, 2))
    assert y.ravel().tolist() == [3, 2] and idx.ravel().tolist() == [1, 0]
    gx = O.maxpool2d_backward(idx, np.array([10, 20], np.float32).reshape(1, 1, 1, 2), 1, 4,
                              (1, 2), (1, 2))
    assert gx.ravel().tolist() == [0, 10, 20, 0]


GEOMS = [  # (H, W, kernel, stride, padding, dilation)
    (112, 112, (3, 3), (2, 2), (1, 1), (1, 1)),   # ResNet stem max pool
    (13, 17, (2, 2), (2, 2), (0, 0), (1, 1)),
    (15, 15, (3, 3), (1, 1), (1, 1), (2, 2)),
    (9, 11, (2, 3), (1, 2), (1, 1), (1, 1)),
    (32, 32, (16, 16), (16, 16), (0, 0), (1, 1)),  # K = 256 taps, the 8-bit limit
]


@pytest.mark.parametrize("geom", GEOMS)
def test_maxpool_matches_torch(geom):
    """Forward values and argmax (first maximum on ties: integer-valued data
    has many) equal torch.nn.functional.max_pool2d(return_indices=True); the
    backward from the 8-bit context equals torch's autograd gradient bit for
    bit (fp32)."""
    H, W, k, s, p, d = geom
    rng = np.random.default_rng(H * 31 + W)
    xa = rng.integers(-4, 5, size=(2, 3, H, W)).astype(np.float32)
    y, idx = O.maxpool2d_forward(xa, k, s, p, d)
    x = torch.from_numpy(xa).requires_grad_(True)
    yt, it = F.max_pool2d(x, k, s, p, d, return_indices=True)
    assert np.array_equal(y, yt.detach().numpy())
    OH, OW = y.shape[2:]
    a, b = idx.astype(np.int64) // k[1], idx.astype(np.int64) % k[1]
    r = np.arange(OH).reshape(1, 1, OH, 1) * s[0] - p[0] + a * d[0]
    c = np.arange(OW).reshape(1, 1, 1, OW) * s[1] - p[1] + b * d[1]
    assert np.array_equal(r * W + c, it.numpy())
    ga = rng.standard_normal(y.shape).astype(np.float32)
    yt.backward(torch.from_numpy(ga))
    gx = O.maxpool2d_backward(idx, ga, H, W, k, s, p, d)
    assert np.array_equal(gx.view(np.uint32), x.grad.numpy().view(np.uint32))
    assert idx.dtype == np.uint8 and idx.size == y.size  # 8 bits per output location


def test_maxpool_bf16_forward():
    rng = np.random.default_rng(1)
    x = torch.from_numpy(rng.standard_normal((2, 4, 20, 20)).astype(np.float32)).to(torch.bfloat16)
    y, idx = O.maxpool2d_forward(bf16_bits(x), (3, 3), (2, 2), (1, 1))
    yt, it = F.max_pool2d(x.float(), 3, 2, 1, return_indices=True)
    assert np.array_equal(y, bf16_bits(yt.to(torch.bfloat16)))


def test_maxpool_rejects_more_than_256_taps():
    x = np.zeros((1, 1, 40, 40), np.float32)
    with pytest.raises(ValueError):
        O.maxpool2d_forward(x, (17, 16), (1, 1))


def test_maxpool_signed_zero_ties_match_torch():
    """Windows whose maximum is a zero of either sign: the oracle stores the
    first zero tap (its sign bit included) and its index, as PyTorch's CPU
    max_pool2d does (update only on a strictly greater value) -- checked bit
    for bit, since -0 == +0 compares equal."""
    rng = np.random.default_rng(5)
    choice = rng.integers(0, 3, size=(2, 3, 16, 18))
    xa = np.where(choice == 0, np.float32(-0.0), np.where(choice == 1, np.float32(0.0),
                                                          np.float32(-1.0))).astype(np.float32)
    y, idx = O.maxpool2d_forward(xa, (3, 3), (2, 2), (1, 1))
    yt, it = F.max_pool2d(torch.from_numpy(xa), 3, 2, 1, return_indices=True)
    assert np.array_equal(y.view(np.uint32), yt.numpy().view(np.uint32))
    bits = y.view(np.uint32)
    assert (bits == 0x80000000).any() and (bits == 0).any()  # both signs win somewhere
