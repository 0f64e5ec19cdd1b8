"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no min/max, no quantisation, no
allocation): only tensor shapes and random value distributions.  It is the one
module both sides of a parity test take their inputs from ("Input
recipe").

Workloads (BASELINE.json configs):
  C1  one fp32 tensor N=4 x D=1024, uniform 2-bit, seed 42 (exact dyadic values)
  C2  ResNet-50 stem activation 256x64x112x112 fp32 (the bn1 input), uniform 2-bit
  C3  ResNet-50 activation set, batch 256, fp32, per-sample {1,2,4,8}, avg 2 bits
  C4  ResNet-152 activation set, batch 1024, bf16, avg 1.25 bits
  C5  ResNet-152 activation set, batch 4096 sharded over k GPUs (bf16, 1.25 bits)

"Activation set": the input of every Conv2d, every
BatchNorm2d and the final Linear of torchvision's ResNet at 224x224 (v1.5:
stride on the 3x3 conv), duplicates counted (a block's conv1 and its
downsample conv each save their own copy).  ReLU masks and max-pool indices are
lossless contexts and are not part of this set.

Value distribution (imitating the heterogeneity of Fig. 3):
  x[n, c, :] = a_n * sigma_c * z + mu_c,  z ~ N(0, 1),
  a_n = exp(zeta_n), sigma_c = exp(zeta_c), zeta ~ N(0, 1), mu_c ~ N(0, 0.1^2);
  inputs of convolutions and of the Linear follow a ReLU, so they are max(0, .)
  (this yields all-zero groups, the R = 0 path); the stem image is N(0, 1);
  bf16 tensors are the RNE of the fp32 draw.
  Data seed of tensor t = 1000 + t; quantiser seed = splitmix64(0xAC7111 ^ t).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

G = 256


@dataclass(frozen=True)
class Act:
    """One saved activation: C channels of H x W (H = W = 1 for the Linear input)."""
    name: str
    C: int
    H: int
    W: int
    relu: bool          # follows a ReLU (conv / linear input) -> non-negative
    image: bool = False  # the raw network input (N(0,1), no channel structure)

    @property
    def D(self) -> int:
        return self.C * self.H * self.W


def _bottleneck_stage(acts: List[Act], prefix: str, in_c: int, width: int, blocks: int,
                      H: int, stride: int) -> int:
    out_c = 4 * width
    for b in range(blocks):
        s = stride if b == 0 else 1
        cin = in_c if b == 0 else out_c
        Ho = H // s
        p = f"{prefix}.{b}"
        acts.append(Act(f"{p}.conv1", cin, H, H, True))
        acts.append(Act(f"{p}.bn1", width, H, H, False))
        acts.append(Act(f"{p}.conv2", width, H, H, True))
        acts.append(Act(f"{p}.bn2", width, Ho, Ho, False))
        acts.append(Act(f"{p}.conv3", width, Ho, Ho, True))
        acts.append(Act(f"{p}.bn3", out_c, Ho, Ho, False))
        if b == 0:
            acts.append(Act(f"{p}.downsample.0", cin, H, H, True))
            acts.append(Act(f"{p}.downsample.1", out_c, Ho, Ho, False))
        H = Ho
    return H


def resnet_activation_set(depth: int) -> List[Act]:
    """Saved activations of torchvision ResNet-50/101/152 at 224x224."""
    blocks = {50: (3, 4, 6, 3), 101: (3, 4, 23, 3), 152: (3, 8, 36, 3)}[depth]
    acts = [Act("conv1", 3, 224, 224, False, image=True), Act("bn1", 64, 112, 112, False)]
    H, in_c = 56, 64
    for li, (width, nb) in enumerate(zip((64, 128, 256, 512), blocks)):
        H = _bottleneck_stage(acts, f"layer{li + 1}", in_c, width, nb, H, 1 if li == 0 else 2)
        in_c = 4 * width
    acts.append(Act("fc", 2048, 1, 1, True))
    return acts


@dataclass(frozen=True)
class Workload:
    name: str
    acts: List[Act]
    N: int
    dtype: str          # "f32" | "bf16"
    avg_bits: Optional[float]   # None => uniform `bits`
    bits: int = 2
    description: str = ""


def workload(name: str, N: Optional[int] = None) -> Workload:
    name = name.lower()
    if name == "c1":
        return Workload("c1", [Act("c1", 1024, 1, 1, False)], 4 if N is None else N, "f32",
                        None, 2, "one fp32 tensor N=4 x 1024, G=256, uniform 2-bit, seed 42")
    if name == "c2":
        return Workload("c2", [Act("bn1", 64, 112, 112, False)], 256 if N is None else N, "f32",
                        None, 2, "ResNet-50 stem activation 256x64x112x112 fp32, uniform 2-bit")
    if name == "c3":
        return Workload("c3", resnet_activation_set(50), 256 if N is None else N, "f32", 2.0,
                        description="ResNet-50 activation set (107 tensors), batch 256, fp32, "
                                    "per-sample {1,2,4,8} averaging 2 bits")
    if name == "c4":
        return Workload("c4", resnet_activation_set(152), 1024 if N is None else N, "bf16", 1.25,
                        description="ResNet-152 activation set (311 tensors), batch 1024, bf16, "
                                    "per-sample {1,2,4,8} averaging 1.25 bits")
    if name == "c5":
        return Workload("c5", resnet_activation_set(152), 4096 if N is None else N, "bf16", 1.25,
                        description="ResNet-152 activation set, batch 4096 sharded over ranks, "
                                    "bf16, averaging 1.25 bits, global allocation")
    raise KeyError(name)


def splitmix64(x: int) -> int:
    """Seed derivation (Steele, Lea, Flood, OOPSLA'14); plumbing, not the method."""
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


def data_seed(t: int) -> int:
    return 1000 + t


def quant_seed(t: int) -> int:
    return splitmix64(0xAC7111 ^ t)


def c1_tensor() -> np.ndarray:
    """C1: x[n, d] = f32(((37 e) mod 101) - 50) * 2^(n-2) / 8, e = n*1024 + d (exact)."""
    N, D = 4, 1024
    e = np.arange(N * D, dtype=np.int64).reshape(N, D)
    base = (((37 * e) % 101) - 50).astype(np.float32)
    scale = np.array([2.0 ** (n - 2) for n in range(N)], np.float32).reshape(N, 1)
    return (base * scale / np.float32(8)).astype(np.float32)


def synth_activation(act: Act, N: int, t: int, dtype: str = "f32", device="cpu",
                     torch=None, out=None):
    """Seeded synthetic activation [N, D] as a torch tensor on `device`, written
    into `out` when given (whole sets are filled without extra copies).  The
    draw is reproducible for the same (act, N, t, dtype, device); the oracle
    side of a parity test receives a host copy of exactly this tensor."""
    if torch is None:
        import torch  # noqa: F811
    g = torch.Generator(device=device)
    g.manual_seed(data_seed(t))
    C, HW = act.C, act.H * act.W
    zeta_n = torch.randn(N, generator=g, device=device)
    zeta_c = torch.randn(C, generator=g, device=device)
    mu_c = 0.1 * torch.randn(C, generator=g, device=device)
    out_dtype = torch.float32 if dtype == "f32" else torch.bfloat16
    if out is None:
        out = torch.empty((N, act.D), dtype=out_dtype, device=device)
    step = max(1, (1 << 28) // max(1, act.D))      # bound temporaries to ~1 GiB fp32
    for lo in range(0, N, step):
        hi = min(N, lo + step)
        z = torch.randn((hi - lo, C, HW), generator=g, device=device)
        if not act.image:
            z.mul_(torch.exp(zeta_n[lo:hi]).view(-1, 1, 1))
            z.mul_(torch.exp(zeta_c).view(1, C, 1))
            z.add_(mu_c.view(1, C, 1))
            if act.relu:
                z.clamp_min_(0.0)
        out[lo:hi].copy_(z.view(hi - lo, -1))
        del z
    return out


def adversarial_tensors(rng: np.random.Generator, D: int = 1024):
    """C1-sized tensors exercising the corner cases of the contract
    (SURVEY §8(d)): constant groups, grid-valued groups, negative minima,
    |Z| >> R, tiny R (degenerate and not), signed zeros, subnormals.
    Returns {name: [N, D] fp32}."""
    out = {}
    N = 4
    out["constant"] = np.full((N, D), 5.0, np.float32)
    k = rng.integers(0, 4, size=(N, D)).astype(np.float32)
    k[:, ::G] = 0.0
    k[:, 1::G] = 3.0
    out["grid_b2"] = (k * np.float32(0.25) - np.float32(7.0)).astype(np.float32)
    out["negative"] = (-np.abs(rng.standard_normal((N, D))) * 3 - 1).astype(np.float32)
    out["large_offset"] = (np.float32(1e4) + rng.random((N, D)).astype(np.float32)).astype(np.float32)
    tiny = np.full((N, D), 1.0, np.float32)
    tiny[0, 5] = np.float32(1.0) + np.float32(2.0 ** -23)
    out["tiny_range"] = tiny
    sub = (rng.random((N, D)) * 2.0 ** -130).astype(np.float32)
    sub[1, :] = np.float32(2.0 ** -100) * rng.random(D).astype(np.float32)
    out["subnormal"] = sub
    # non-degenerate tiny ranges (SURVEY §8(d) "R in {2^-100, 2^-90}", reading
    # 16's threshold R < 2^-96): every group spans [0, R] exactly with R = 2^-95,
    # 2^-90, 2^-96 (the smallest non-degenerate range) and the largest float
    # below 2^-96 (degenerate: all codes 0); a third of the members are
    # subnormal, a third normal in (0, R), a third zero, so inv14 is near
    # B 2^110 and the codes are non-zero
    tr = np.zeros((N, D), np.float32)
    k = np.arange(D)
    for n, R in enumerate((np.float32(2.0 ** -95), np.float32(2.0 ** -90),
                           np.float32(2.0 ** -96),
                           np.nextafter(np.float32(2.0 ** -96), np.float32(0)))):
        u = (rng.random(D) * float(R)).astype(np.float32)
        s = (rng.random(D) * 2.0 ** -126).astype(np.float32)
        tr[n] = np.where(k % 3 == 0, u, np.where(k % 3 == 1, s, np.float32(0)))
        tr[n, 0::G] = 0.0
        tr[n, 1::G] = R
    out["tiny_range_nondegenerate"] = tr
    z = np.zeros((N, D), np.float32)
    z[:, 1::2] = -0.0
    z[2, 7] = 1.0
    out["signed_zero"] = z
    out["normal"] = rng.standard_normal((N, D)).astype(np.float32)
    return out


def expected_counts():
    """Per-sample element counts of the activation sets."""
    return {50: (107, 21_778_432), 152: (311, 44_658_688)}


def bytes_per_elem(dtype: str) -> int:
    return 4 if dtype == "f32" else 2


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def total_elements(acts: List[Act], N: int) -> int:
    return N * sum(a.D for a in acts)


def mean(xs):
    return math.fsum(xs) / max(1, len(xs))
